make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1
export DHZ_GUIDED_PATH=twopass
ncu --section LaunchStats --section Occupancy --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k "regex:k_gx" -c 2 python tools/guided_once.py > gpurun_out/occ.log 2>&1
grep -E 'k_gx|Duration|Registers|Shared Memory|Block Limit|Achieved Occupancy|Theoretical Occ|inst_executed|Waves' gpurun_out/occ.log
