#!/bin/bash
# Builds the overlap probe against the package's object files.
cd "$(dirname "$0")"
make -C ../../paper_2512_16609_b200/csrc -j16 > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include overlap_probe.cu \
  ../../paper_2512_16609_b200/csrc/build/*.o -o overlap_probe
