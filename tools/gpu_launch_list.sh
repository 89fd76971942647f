# ncu launch list (per-kernel duration + DRAM bytes) of tools/guided_once.py
mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
export DHZ_GUIDED_PATH=${DHZ_GUIDED_PATH:-twopass} C5N=${C5N:-8} REPS=1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ll.csv python tools/guided_once.py > gpurun_out/ll.log 2>&1
python tools/summarize_launches.py gpurun_out/ll.csv
