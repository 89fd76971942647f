#!/bin/bash
# Build-flag variants of the library, each timed on the default bench (C3).
# usage: VARIANTS="-DFOO=1;-DFOO=2" bash tools/variant_bench.sh [bench args]
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "" "${VS[@]}"; do
  make -C paper_2512_16609_b200/csrc clean > /dev/null
  make -C paper_2512_16609_b200/csrc -j16 NVFLAGS_EXTRA="$v" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  r=$(python bench.py --no-cpu-baseline --e2e-steps 0 --steps 20 "$@" | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['pipeline_roofline']['stage_ms'])")
  echo "variant [$v]: $r"
done
