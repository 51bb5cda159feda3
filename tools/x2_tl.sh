WQB200_LIB=tools/_build/libwqb200_tl.so python tools/x2_tl.py
W_IK1=0 WQB200_LIB=tools/_build/libwqb200_tl.so python tools/x2_tl.py
