mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_api_gpu.py tests/test_frameio.py tests/test_multi_gpu.py -x -q 2>&1 | tail -1
for c in ${CFGS:-c1 c2}; do
  python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/bps_$c.json 2> /dev/null
  python - "$c" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/bps_{sys.argv[1]}.json").read().strip().splitlines()[-1])
e = d["e2e"]
print(sys.argv[1], "e2e", e["value"], "process_stream", e["process_stream"]["value"], e["process_stream"]["ms_per_step"])
PY
done
