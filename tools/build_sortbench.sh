#!/bin/sh
# Build the depth-sort A/B harness (tools/sortbench.cu) against the library objects.
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2412_03378_b200 import build as b; b.build()"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -Ipaper_2412_03378_b200/csrc \
  tools/sortbench.cu build/csrc/vg_radix.o -o build/sortbench
