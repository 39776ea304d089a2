#!/bin/bash
# Profiling variant of the engine: parity.cu with -DAP_SAMPLE_TRACE (stage clocks of the PER
# sampler), linked with the other in-tree objects; load it with AP_LIB_PATH=/tmp/libtrace.so.
set -e
cd "$(dirname "$0")/../../paper_2007_04069_b200"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I../include -fmad=false \
  -DAP_SAMPLE_TRACE -c csrc/parity.cu -o /tmp/parity_trace.o
objs=$(ls _build/*.o | grep -v parity.cu.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/libtrace.so $objs /tmp/parity_trace.o
