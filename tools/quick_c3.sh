#!/bin/bash
# Quick GPU check of the C3 video path: build, the video parity tests, one bench
# line (stage times), and the ncu launch list of the bench command.
mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest ${TESTS:-tests/test_video_gpu.py tests/test_fullsize_gpu.py tests/test_golden_gpu.py} -x -q > gpurun_out/pt.log 2>&1
tail -2 gpurun_out/pt.log
python bench.py --no-cpu-baseline --e2e-steps 0 --steps ${STEPS:-20} ${BENCH_ARGS} > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_q.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["value"], d["pipeline_roofline"]["frac"], d["pipeline_roofline"]["stage_ms"], d["clocks"])
PY
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "regex:k_" --csv --log-file gpurun_out/launches_q.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_q.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_q.csv
