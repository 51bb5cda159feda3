# per-CTA phase clocks of x2 (tools build) and plain timings
WQB200_LIB=tools/_build/libwqb200_tl.so python tools/x2_tl.py
python tools/x2_time.py
