for rep in 1 2; do
for cfg in medium opaque; do
  (cd abtmp/head && python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-facade --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg head', d['value'], d['ms_per_step'])")
  for r in 1.0 1.5 2.0; do
    VG_SEG_RATIO=$r python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu --no-facade --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg ratio$r', d['value'], d['ms_per_step'])"
  done
done
done
