# round 2, GPU call 2: the fused 3-D engine's parity first, then the GPU suite
# and a quick config 4 bench + the DMMA occupancy microbenchmark
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KFVM_DEBUG_SYNC=${KFVM_DEBUG_SYNC:-0}
timeout 900 python -m pytest tests/test_fused3.py -x -q -p no:cacheprovider > gpurun_out/pytest_fused3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused3.log
timeout 1800 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --steps 5 > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 600 python bench.py --no-cpu --config 3 --steps 5 > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench/dmma_occupancy.cu -o /tmp/dmma_occ && timeout 300 /tmp/dmma_occ > gpurun_out/dmma_occupancy.txt 2>&1
ls -la gpurun_out
