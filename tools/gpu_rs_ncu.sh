mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
ncu --set full --import-source on --clock-control none -k "regex:${KREGEX:-k_rs_}" -c ${NK:-3} -o gpurun_out/rs_full \
    python bench.py --config c3d --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/rs_ncu.log 2>&1
tail -2 gpurun_out/rs_ncu.log
