cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_kx3.csv python bench.py --config 3 --steps 1 --warmup 3 --no-cpu --kxrcf > gpurun_out/ncu_l3.log 2>&1; tail -1 gpurun_out/ncu_l3.log | cut -c1-80
