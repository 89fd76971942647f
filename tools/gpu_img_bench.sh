# full GPU suite, then the image-mode bench lines
mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_gpu.log 2>&1; tail -2 gpurun_out/pt_gpu.log
python bench.py --config c2 --steps 10 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config c5 --steps 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c2 c5; do python - "$c" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["ms_per_step"], d["pipeline_roofline"]["frac"], d["pipeline_roofline"]["stage_ms"], d["roofline"]["frac"], d["e2e"]["value"], d["clocks"]["sm_mhz"])
PY
done
