# round 2, GPU call 1: GPU tests, the default bench (config 4, 512^3), the
# reference arm, the launch list and one ncu --set full capture of the 3-D
# reconstruction kernel at 512^3 (run from the repo root on the GPU box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/box.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/profile_step.py --config 4 --steps 1 > gpurun_out/ncu_l.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_states_u -s 2 -c 1 -o gpurun_out/prof_c4_states python tools/profile_step.py --config 4 --steps 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
