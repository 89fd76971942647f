# C1 latency A/B: small-batch K1 tiles (DHZ_K1_BH=16 vs 64) and the direct K6 (DHZ_K6_DIRECT=1 vs 0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_video_gpu.py tests/test_golden_gpu.py tests/test_api_gpu.py -x -q 2>&1 | tail -2
for v in "64 0" "16 0" "64 1" "16 1" "default"; do
  set -- $v
  if [ "$1" = default ]; then unset DHZ_K1_BH DHZ_K6_DIRECT; else export DHZ_K1_BH=$1 DHZ_K6_DIRECT=$2; fi
  for c in c1 ${EXTRA}; do
  python bench.py --config $c --steps 20 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', d['config']['workload'][:3], d['ms_per_step'], d['pipeline_roofline']['stage_ms'])"
  done
done
unset DHZ_K1_BH DHZ_K6_DIRECT
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_" --csv --log-file gpurun_out/launches_c1.csv \
    python bench.py --config c1 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_c1.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_c1.csv
