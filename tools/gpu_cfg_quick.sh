# build, optional tests ($TESTS), bench lines for $CFGS (no e2e / cpu baseline)
mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest $TESTS -x -q > gpurun_out/pt_q.log 2>&1; tail -1 gpurun_out/pt_q.log; fi
for c in ${CFGS:-c3}; do
  python bench.py --config $c --steps ${STEPS:-10} --e2e-steps 0 --no-cpu-baseline > gpurun_out/bq_$c.json 2> gpurun_out/bq_$c.err
  python - "$c" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/bq_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], d["ms_per_step"], d["value"], d["pipeline_roofline"]["frac"], d["pipeline_roofline"]["stage_ms"], d["clocks"]["sm_mhz"], d["roofline"]["frac"])
PY
done
