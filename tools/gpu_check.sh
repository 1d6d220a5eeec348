#!/bin/bash
# quick GPU iteration: parity tests + per-config bench summaries
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-2 1 3}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu ${BENCH_ARGS} > gpurun_out/bench_c$c.log 2>&1
  tail -1 gpurun_out/bench_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:40], '%.3e'%d['value'], 'frac=%.3f'%d['roofline']['frac'], {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})" 2>&1 | tail -1
done
