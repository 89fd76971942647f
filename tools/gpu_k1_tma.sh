#!/bin/bash
# K1 with TMA-staged rows (DHZ_K1_TMA=1) against the LDG default: video parity tests
# under the TMA variant, then C3 / C4 / C1 bench lines for both.
mkdir -p gpurun_out
DHZ_K1_TMA=1 timeout 900 python -m pytest tests/test_video_gpu.py tests/test_fullsize_gpu.py tests/test_golden_gpu.py tests/test_memory_safety_gpu.py -x -q > gpurun_out/pt_tma.log 2>&1
tail -3 gpurun_out/pt_tma.log
for t in 0 1; do
  for c in c3 c4 c1; do
    r=$(DHZ_K1_TMA=$t timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 0 --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['pipeline_roofline']['stage_ms'])")
    echo "DHZ_K1_TMA=$t $c: $r"
  done
done 2>&1 | tee gpurun_out/k1_tma.txt
