# Round-2 evidence pass on the GPU box (outputs under gpurun_out/; the files
# judged are copied to profiles/):  bash tools/evidence_r2.sh
#   GPU tests, smoke, the checking-build run (debug_checks), bench lines of
#   configs 3/2/4/5 + deterministic config 3, the opaque launch-balance log
#   (walk_stats, profiling build) and an ncu --set full capture of a
#   segmented opaque backward.
python -m pytest tests -x -q -m gpu > gpurun_out/ev_tests.log 2>&1; echo tests=$? > gpurun_out/ev_status.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo smoke=$? >> gpurun_out/ev_status.log
python tools/debug_checks.py --out gpurun_out/debug_checks_r2.md > gpurun_out/ev_debug.log 2>&1; echo debug=$? >> gpurun_out/ev_status.log
for c in large medium opaque tomography; do python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2_bench_$c.json 2> gpurun_out/ev_bench_$c.err; echo bench_$c=$? >> gpurun_out/ev_status.log; done
python bench.py --config large --steps 5 --warmup 3 --deterministic > gpurun_out/r2_bench_large_deterministic.json 2> gpurun_out/ev_bench_det.err; echo bench_det=$? >> gpurun_out/ev_status.log
python tools/walk_stats.py opaque --views 0,3,7 > gpurun_out/ev_walk_opaque.log 2>&1; echo walk=$? >> gpurun_out/ev_status.log
ncu --set full --clock-control none --import-source on -k regex:k_render_bwd --launch-skip 3 --launch-count 1 -o gpurun_out/prof_r2_opaque_seg python tools/profile_view.py --config opaque --views 4 > gpurun_out/ev_ncu.log 2>&1; echo ncu=$? >> gpurun_out/ev_status.log
