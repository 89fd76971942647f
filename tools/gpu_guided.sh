mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 python tools/guided_probe.py c5 c2 c5nb > gpurun_out/gprobe.log 2>&1; cat gpurun_out/gprobe.log | tail -20
timeout 1200 python -m pytest tests/test_image_gpu.py tests/test_c5_gpu.py tests/test_golden_gpu.py -x -q > gpurun_out/pt_img.log 2>&1; tail -30 gpurun_out/pt_img.log
