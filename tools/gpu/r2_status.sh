# round 2 re-entry: where does HEAD stand on the GPU (fused 3-D engine parity,
# the GPU suite incl. the stated-config gate, config 3/4 timing, reference arm)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nproc; lscpu | grep -E "Model name|^CPU\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/box.txt 2>&1
timeout 900 python -m pytest tests/test_fused3.py -x -q -p no:cacheprovider > gpurun_out/pytest_fused3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused3.log
out=gpurun_out/quick.txt; : > $out
timeout 300 python tools/time_step.py --config 3 >> $out 2>&1
timeout 300 python tools/time_step.py --config 3 --opt engine=2 >> $out 2>&1
timeout 300 python tools/time_step.py --config 4 --steps 2 >> $out 2>&1
timeout 300 python tools/time_step.py --config 4 --steps 2 --opt engine=2 >> $out 2>&1
timeout 900 python bench.py --no-cpu --steps 5 > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
ls -la gpurun_out
