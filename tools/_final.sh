cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | cut -c1-200
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-200
for c in 1 3; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c$c.log 2>&1; tail -1 gpurun_out/bench_c$c.log | cut -c1-150; done
python bench.py --config 4 --n 256 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4_256.log 2>&1
python bench.py --config 5 --n 256 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c5_256.log 2>&1
python bench.py --config 4 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c4_full.log 2>&1
python bench.py --config 5 --n 1024 --nz 128 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c5_block.log 2>&1
for c in 2 3; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu --kxrcf > gpurun_out/bench_c${c}_kx.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config 3 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_l3.log 2>&1
