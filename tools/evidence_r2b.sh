# Round-2 evidence, part 2: the parity margins report and the config-3 ncu launch list
# (cold, serialised per-launch times of the same command as the bench's step).
python tools/parity_report.py > gpurun_out/ev_parity.log 2>&1; echo parity=$? > gpurun_out/ev2_status.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_large_3views.csv python tools/profile_view.py --config large --views 3 > gpurun_out/ev_launch.log 2>&1; echo launches=$? >> gpurun_out/ev2_status.log
