#!/bin/bash
# incremental build (tools only): compile the .cu files that changed, in parallel, and link
# paper_1703_10016_b200/libwqb200.so (or $1).  __graft_entry__.build() is the reference build.
set -u; TAG=${TAG:-}; EXTRA=${EXTRA:-}
cd "$(dirname "$0")/.."
OUT=${1:-paper_1703_10016_b200/libwqb200.so}
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include $EXTRA"
mkdir -p build/obj$TAG
pids=()
for f in paper_1703_10016_b200/csrc/*.cu; do
  o=build/obj$TAG/$(basename "$f" .cu).o
  if [ ! -f "$o" ] || [ "$f" -nt "$o" ] || [ -n "$(find paper_1703_10016_b200/csrc include -name '*.cuh' -newer "$o" -o -name '*.h' -newer "$o")" ]; then
    nvcc $FLAGS -c "$f" -o "$o" 2>&1 | grep -v "^$" &
    pids+=($!)
  fi
done
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o "$OUT" build/obj$TAG/*.o
echo "linked $OUT"
