#!/bin/bash
# Round-2 refresh on the GPU box: full GPU suite + smoke, every bench config, the
# reference arm, ncu launch lists (C3, C4, C5) and --set full captures of the top kernels.
set -x
mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pt_gpu.log 2>&1; tail -2 gpurun_out/pt_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -5 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
for c in c1 c2 c4 c3d; do
  python bench.py --config $c --steps 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --config c5 --steps 3 --e2e-steps 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c3.json 2> gpurun_out/bench_ref.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none -k "regex:k_" --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --metrics $M --clock-control none -k "regex:k_" --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --config c4 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_c4.log 2>&1
ncu --metrics $M --clock-control none -k "regex:k_" --csv --log-file gpurun_out/launches_c5.csv \
    python bench.py --config c5 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_c5.log 2>&1
ncu --metrics $M --clock-control none -k "regex:k_" --csv --log-file gpurun_out/launches_c3d.csv \
    python bench.py --config c3d --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_c3d.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_(dark_rows|recover_lut_diag)" -c 2 \
    -o gpurun_out/full_c3 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_(gx_ab|gx_out|gf_apply2)" -c 3 \
    -o gpurun_out/full_c5 python bench.py --config c5 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_c5.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_(balance_band|build_g)" -c 2 \
    -o gpurun_out/full_c4_balance python bench.py --config c4 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_rs_" -c 3 \
    -o gpurun_out/full_c3d python bench.py --config c3d --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_c3d.log 2>&1
echo done
