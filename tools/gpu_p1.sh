# pass-1 form A/B (DHZ_PASS1=gx|gy): fused/two-pass tests, probe timings, launch list
mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_guided_fused_gpu.py tests/test_c5_gpu.py -x -q > gpurun_out/pt_p1.log 2>&1; tail -1 gpurun_out/pt_p1.log
for p in gx gy; do DHZ_PASS1=$p PATHS=twopass C5N=8 python tools/guided_probe.py c5nb c5 > gpurun_out/gp_$p.log 2>&1; echo $p; cat gpurun_out/gp_$p.log; done
DHZ_PASS1=gy bash tools/gpu_launch_list.sh 2>&1 | grep 'k_g'
