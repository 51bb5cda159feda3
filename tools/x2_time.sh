for v in 4 3; do echo "v$v"; WQB200_X2=$v python tools/x2_time.py; done
