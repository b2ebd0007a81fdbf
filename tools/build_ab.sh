#!/bin/bash
# Build library variants for tools/ab_bench.sh:
#   [FILE="vg_blend.cu [vg_x.cu ...]"] [KEEP="build/csrc/x.o ..."] tools/build_ab.sh name "-DVG_FWD_MINB=8 ..." [name2 "flags2" ...]
# Every file in FILE is recompiled with the variant's flags; the other objects
# come from the regular build.
set -e
cd "$(dirname "$0")/.."
python -c "from paper_2412_03378_b200 import build as b; b.build()"
mkdir -p build/ab
ARCH="-gencode arch=compute_100a,code=sm_100a"
FILE=${FILE:-vg_blend.cu}
objs=$(ls build/csrc/*.o)
for f in $FILE; do
  # every unit built from this source (vg_blend.cu -> vg_blend.o, vg_blend_fwd.o)
  objs=$(echo "$objs" | grep -v "/${f%.cu}\(_[a-z]*\)\?\.o")
done
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  vobjs=""
  for f in $FILE; do
    o=build/ab/${name}_${f%.cu}.o
    nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -Iinclude \
      -Ipaper_2412_03378_b200/csrc $flags $EXTRA -c paper_2412_03378_b200/csrc/$f -o $o \
      -Xptxas -v 2>&1 | grep -E "registers" | head -4 | sed "s/^/$name: /"
    vobjs="$vobjs $o"
  done
  nvcc $ARCH -shared -cudart static -o build/ab/$name.so $objs $vobjs $KEEP
done
