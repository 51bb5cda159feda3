python tools/x2_time.py
