mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
export DHZ_GUIDED_PATH=${DHZ_GUIDED_PATH:-twopass}
python tools/guided_once.py || exit 1
export C5N=${C5N:-8} REPS=1
ncu --set full --import-source on --clock-control none -k "regex:${KREGEX:-k_gx}" -c ${NK:-2} -o gpurun_out/gx_full python tools/guided_once.py > gpurun_out/gx_ncu.log 2>&1
tail -3 gpurun_out/gx_ncu.log
