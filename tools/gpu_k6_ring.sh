# K6 bulk-copy ring (DHZ_K6_RING=1) vs the LDG form: parity tests with the ring forced on
# every vectorised launch, then C3 / C4 timings of both.
mkdir -p gpurun_out
DHZ_K6_RING=1 DHZ_K6_DIRECT=0 timeout 900 python -m pytest tests/test_video_gpu.py tests/test_golden_gpu.py tests/test_memory_safety_gpu.py -x -q -k "not tiles_every_radius" 2>&1 | tail -2
DHZ_K6_RING=1 timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_fuzz_gpu.py -x -q 2>&1 | tail -2
for v in 0 1 0 1; do
  export DHZ_K6_RING=$v
  for c in c3 c4; do
  python bench.py --config $c --steps 20 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('ring=$v', d['config']['workload'][:3], d['ms_per_step'], d['pipeline_roofline']['stage_ms'])"
  done
done
