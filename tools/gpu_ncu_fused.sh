mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
export C5N=${C5N:-2} PATHS=fused
python tools/guided_probe.py ${CFG:-c5nb} > gpurun_out/gprobe_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_gf_fused -s ${SKIP:-1} -c 1 -o gpurun_out/${OUT:-fused} \
  python tools/guided_probe.py ${CFG:-c5nb} > gpurun_out/ncu_fused.log 2>&1
tail -3 gpurun_out/ncu_fused.log; cat gpurun_out/gprobe_plain.log
