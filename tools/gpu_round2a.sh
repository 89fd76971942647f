set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_gpu.log 2>&1; tail -3 gpurun_out/pt_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -5 gpurun_out/smoke.log
bash tools/round_profiles.sh > gpurun_out/rp.log 2>&1
for f in gpurun_out/bench_*.json; do echo $f; tail -c 600 $f; echo; done
