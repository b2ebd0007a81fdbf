#!/bin/bash
# A/B library variants abtmp/ab/<name>.so (+ abtmp/head, a built copy of the
# previous commit): serial per-kernel times and the overlapped step.
#   CFGS="large" VARIANTS="noseg:VG_SEG_BWD=0 full:VG_SEG_BWD=1" tools/ab_libs.sh
cfgs=${CFGS:-large}
lib=paper_2412_03378_b200/libvolgauss_b200.so
cp $lib /tmp/lib_orig.so
one() {  # dir label env...
  dir=$1; label=$2; shift 2
  (cd $dir && env "$@" VG_OVERLAP=0 python bench.py --config $cfg --views 16 --steps 3 --no-e2e --no-cpu 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$cfg $label serial', d['ms_per_step'], {n: round(x['ms_per_step'], 3) for n, x in k.items() if n.startswith('render')})")
  (cd $dir && env "$@" python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $label step', d['ms_per_step'])")
}
for rep in 1 2; do
for cfg in $cfgs; do
  [ -d abtmp/head ] && one abtmp/head head X=1
  for v in $VARIANTS; do
    name=${v%%:*}; envs=${v#*:}
    cp abtmp/ab/$name.so $lib
    one . $name $envs
  done
  cp /tmp/lib_orig.so $lib
done
done
