#!/bin/bash
# tools-only build of the library with the x2 per-CTA phase clocks (WQ_X2_TIMELINE)
cd "$(dirname "$0")/.." && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -DWQ_X2_TIMELINE -I include -o tools/_build/libwqb200_tl.so \
  paper_1703_10016_b200/csrc/*.cu
