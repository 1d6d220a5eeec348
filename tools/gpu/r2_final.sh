# round 2 final evidence at HEAD: full GPU suite, default bench (config 4) +
# reference arm, configs 2/3/5 bench lines, config 4 launch list, ncu --set
# full of the 3-D reconstruction kernel (k_states_w) at 512^3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nproc; lscpu | grep -E "Model name|^CPU\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/box.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rfxX > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
timeout 600 python bench.py --config 2 --no-cpu > gpurun_out/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2.log
timeout 600 python bench.py --config 3 --no-cpu > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
timeout 900 python bench.py --config 5 --no-cpu > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/profile_step.py --config 4 --steps 1 > gpurun_out/ncu_l.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_states_w -s 2 -c 1 -o gpurun_out/prof_c4_states_w python tools/profile_step.py --config 4 --steps 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
