# one compute-sanitizer tool per gpurun call (TOOL=memcheck|racecheck|synccheck|initcheck)
mkdir -p gpurun_out
make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1 || { echo build failed; exit 1; }
python tools/sanitize_cases.py > gpurun_out/san_plain_${TOOL}.log 2>&1 || { echo plain run failed; tail gpurun_out/san_plain_${TOOL}.log; exit 1; }
timeout 2400 compute-sanitizer --tool ${TOOL} --target-processes all --print-limit 50 python tools/sanitize_cases.py \
  > gpurun_out/sanitizer_${TOOL}.log 2>&1
echo "exit $?"; tail -5 gpurun_out/sanitizer_${TOOL}.log
