cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config 5 --n 256 --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c5_256.log 2>&1
grep '^{' gpurun_out/bench_c5_256.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['whole_step_fp64_frac'], d['kernel_ms_per_step'])
"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_256.csv python tools/profile_step.py --config 5 --n 256 --steps 1 > gpurun_out/ncu_l5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_states_u -s 2 -c 1 -o gpurun_out/prof_c5_256_states python tools/profile_step.py --config 5 --n 256 --steps 1 > gpurun_out/ncu_f5.log 2>&1
tail -2 gpurun_out/ncu_f5.log
