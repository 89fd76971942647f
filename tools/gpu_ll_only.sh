mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest ${TESTS:-tests/test_guided_fused_gpu.py} -x -q > gpurun_out/pt_ll.log 2>&1; tail -1 gpurun_out/pt_ll.log
bash tools/gpu_launch_list.sh 2>&1 | grep 'k_g'
