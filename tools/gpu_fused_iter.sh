# quick iteration on the fused guided kernel: build, parity probe vs the strip path, tests, ncu
mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
C5N=8 timeout 600 python tools/guided_probe.py c5 c5nb c2 > gpurun_out/gprobe.log 2>&1; cat gpurun_out/gprobe.log | tail -5
timeout 900 python -m pytest tests/test_image_gpu.py tests/test_c5_gpu.py tests/test_golden_gpu.py -x -q > gpurun_out/pt_img.log 2>&1; tail -3 gpurun_out/pt_img.log
if [ -n "$NCU" ]; then
  export C5N=2 PATHS=fused
  ncu --set full --import-source on --clock-control none -k regex:k_gf_fused -s 1 -c 1 -o gpurun_out/${OUT:-fused} \
    python tools/guided_probe.py ${CFG:-c5nb} > gpurun_out/ncu_fused.log 2>&1; tail -2 gpurun_out/ncu_fused.log
fi
