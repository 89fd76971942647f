#!/bin/bash
# Round-end measurements on the GPU box: bench lines for every config, the ncu
# launch list of the default bench command, and one --set full capture of the
# two big video kernels.  Everything lands in gpurun_out/ (copied to profiles/).
set -x
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
for c in c1 c2 c4 c3d; do
  python bench.py --config $c --steps 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --config c5 --steps 3 --e2e-steps 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c3.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "regex:k_" --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_(dark_rows|recover_lut_diag)" -c 2 \
    -o gpurun_out/full_c3 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
    > gpurun_out/ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k "regex:k_" --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --config c4 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_c4.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_(balance_band|build_g)" -c 2 \
    -o gpurun_out/full_c4_balance python bench.py --config c4 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline \
    > gpurun_out/ncu_full_c4.log 2>&1
echo done
