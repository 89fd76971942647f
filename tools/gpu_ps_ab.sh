# process_stream A/B on one box: staging-copy outputs + immediate input copies (old) vs
# pinned per-frame outputs + deferred parallel input copies (new)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_api_gpu.py tests/test_frameio.py tests/test_multi_gpu.py -x -q 2>&1 | tail -3
for c in ${CFGS:-c3 c4 c1}; do
  for mode in old new old new; do
    if [ $mode = old ]; then export DHZ_PINNED_OUT_BYTES=0 DHZ_PS_LAZY=0; else unset DHZ_PINNED_OUT_BYTES DHZ_PS_LAZY; fi
    python bench.py --config $c --steps 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bps_${c}_$mode.json 2> /dev/null
    python - "$c" "$mode" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/bps_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
e = d["e2e"]
print(sys.argv[1], sys.argv[2], "e2e", e["value"], "process_stream", e["process_stream"]["value"], e["process_stream"]["ms_per_step"])
PY
  done
done
