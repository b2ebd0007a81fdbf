#!/bin/bash
# A/B the blend kernels of several prebuilt library variants (build/ab/*.so)
# with serial per-kernel timing (VG_OVERLAP=0); run on the GPU box:
#   tools/ab_bench.sh [views] [steps] [config]
views=${1:-16}; steps=${2:-3}; config=${3:-large}
lib=paper_2412_03378_b200/libvolgauss_b200.so
cp $lib /tmp/lib_orig.so
for v in build/ab/*.so; do
  cp $v $lib
  for rep in 1 2; do
    VG_OVERLAP=0 python bench.py --config $config --views $views --steps $steps --no-e2e --no-cpu $BENCH_ARGS 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$v', d['ms_per_step'], {n: round(x['ms_per_step'], 3) for n, x in k.items() if isinstance(x, dict)})"
  done
done
cp /tmp/lib_orig.so $lib
