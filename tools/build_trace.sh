#!/bin/bash
# Builds tools/lu_trace: the library compiled with -DSAP_LU_TRACE plus a driver that prints the LU phase timeline.
set -e
cd "$(dirname "$0")/.."
mkdir -p /tmp/trbuild
for f in paper_1509_07919_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSAP_LU_TRACE -DSAP_SWEEP_TRACE -Iinclude -Ipaper_1509_07919_b200/csrc \
       -Xcompiler -fPIC -c "$f" -o /tmp/trbuild/$(basename "$f").o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude tools/lu_trace.cu /tmp/trbuild/*.o -o tools/lu_trace -lcudart_static

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude tools/sweep_trace.cu /tmp/trbuild/*.o -o tools/sweep_trace -lcudart_static
