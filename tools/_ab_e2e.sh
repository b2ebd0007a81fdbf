# value / ms / e2e per variant (with e2e), config medium + large serial finalize
lib=paper_2412_03378_b200/libvolgauss_b200.so
cp $lib /tmp/lib_orig.so
one() { dir=$1; label=$2; cfg=$3
  (cd $dir && python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-facade 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $label', d['value'], d['ms_per_step'], d['e2e']['value'], round(d['kernels']['finalize']['ms_per_step'],3))")
}
for rep in 1 2; do
for cfg in medium large; do
  one abtmp/head head $cfg
  for v in base lazy; do cp abtmp/ab/$v.so $lib; one . $v $cfg; done
  cp /tmp/lib_orig.so $lib
done
done
