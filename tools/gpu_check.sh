set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv > gpurun_out/gpu.txt
free -g >> gpurun_out/gpu.txt; nproc >> gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_gpu.log 2>&1; tail -3 gpurun_out/pt_gpu.log
timeout 900 python tools/c5_probe.py --full > gpurun_out/c5_probe.log 2>&1; tail -8 gpurun_out/c5_probe.log
