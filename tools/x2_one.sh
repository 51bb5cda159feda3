WQB200_LIB=tools/_build/libwqb200_one.so python tools/x2_tl.py
WQB200_LIB=tools/_build/libwqb200_tl.so python tools/x2_tl.py
