# loopback multi-rank tests, the one-rank NCCL path (now graph-captured), FP64 latencies
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_loopback.py tests/test_nccl_one_rank.py tests/test_handles.py -x -q -p no:cacheprovider -rf > gpurun_out/pytest_loop.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_loop.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench/fp64_latency.cu -o /tmp/lat && timeout 60 /tmp/lat > gpurun_out/fp64_latency.txt 2>&1
tail -30 gpurun_out/pytest_loop.log; cat gpurun_out/fp64_latency.txt
