# k_gw_sums A/B (DHZ_GW_BF=0 vs default) on C5 frames + image-mode parity tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_image_gpu.py tests/test_c5_gpu.py tests/test_golden_gpu.py tests/test_guided_fused_gpu.py -x -q 2>&1 | tail -2
for v in 0 1 0 1; do
  export DHZ_GW_BF=$v
  for c in c5 c2; do
  python bench.py --config $c --steps 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('bf=$v', d['config']['workload'][:3], d['ms_per_step'], d['pipeline_roofline']['stage_ms'])"
  done
done
unset DHZ_GW_BF
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_g" --csv --log-file gpurun_out/launches_gw.csv \
    python bench.py --config c5 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_gw.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_gw.csv
