cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_l.log 2>&1; tail -1 gpurun_out/ncu_l.log | cut -c1-100
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config 3 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_l3.log 2>&1; tail -1 gpurun_out/ncu_l3.log | cut -c1-100
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage_row -s 3 -c 1 -o gpurun_out/prof_c2_states python tools/profile_step.py --config 2 --steps 2 > gpurun_out/ncu1.log 2>&1; tail -1 gpurun_out/ncu1.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flux -s 3 -c 1 -o gpurun_out/prof_c2_flux python tools/profile_step.py --config 2 --steps 2 > gpurun_out/ncu2.log 2>&1; tail -1 gpurun_out/ncu2.log
