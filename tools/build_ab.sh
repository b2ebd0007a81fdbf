#!/bin/bash
# Build library variants of the blend kernels for tools/ab_bench.sh:
#   [FILE=vg_blend.cu] tools/build_ab.sh name "-DVG_FWD_MINB=8 ..." [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2412_03378_b200 import build as b; b.build()"
mkdir -p build/ab
ARCH="-gencode arch=compute_100a,code=sm_100a"
FILE=${FILE:-vg_blend.cu}
base=${FILE%.cu}
objs=$(ls build/csrc/*.o | grep -v "/$base.o")
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -Iinclude \
    -Ipaper_2412_03378_b200/csrc $flags $EXTRA -c paper_2412_03378_b200/csrc/$FILE -o build/ab/$name.o \
    -Xptxas -v 2>&1 | grep -E "registers" | head -4 | sed "s/^/$name: /"
  nvcc $ARCH -shared -cudart static -o build/ab/$name.so $objs build/ab/$name.o
done
