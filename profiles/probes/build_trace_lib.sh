#!/bin/bash
# Profiling variant of the engine: parity.cu with -DAP_SAMPLE_TRACE (stage clocks of the PER
# sampler) and fused_mlp.cu with -DAP_FUSED_TILE_TRACE (stage stamps of CTA 0's tiles), linked
# with the other in-tree objects; load it with AP_LIB_PATH=/tmp/libtrace.so.
set -e
cd "$(dirname "$0")/../../paper_2007_04069_b200"
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I../include"
nvcc $F -fmad=false -DAP_SAMPLE_TRACE -c csrc/parity.cu -o /tmp/parity_trace.o
nvcc $F -DAP_FUSED_TILE_TRACE -c csrc/fused_mlp.cu -o /tmp/fused_trace.o
objs=$(ls _build/*.o | grep -v -e parity.cu.o -e fused_mlp.cu.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/libtrace.so $objs /tmp/parity_trace.o /tmp/fused_trace.o
