#!/bin/bash
# Re-entry check on the GPU box: full GPU suite, smoke, every bench config.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt_gpu.log 2>&1; tail -3 gpurun_out/pt_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 600 gpurun_out/bench_c3.json
for c in c1 c2 c4 c3d; do
  python bench.py --config $c --steps 10 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --config c5 --steps 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo done
