# two-pass exact guided filter: parity tests, then timings of the three image-mode forms
mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest ${TESTS:-tests/test_guided_fused_gpu.py} -x -q > gpurun_out/pt_tp.log 2>&1; tail -3 gpurun_out/pt_tp.log
PATHS=${PATHS:-strip,fused,twopass} C5N=${C5N:-8} timeout 600 python tools/guided_probe.py ${CFGS:-c5nb c5 c2} > gpurun_out/gprobe.log 2>&1; cat gpurun_out/gprobe.log | tail -5
