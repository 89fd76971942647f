make -C paper_2512_16609_b200/csrc -j16 > /dev/null 2>&1
for pdl in 1 0 1 0; do
 for c in c3 c1; do
  DHZ_PDL=$pdl python bench.py --config $c --steps 20 --e2e-steps 0 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('pdl=$pdl', '$c', d['ms_per_step'], d['pipeline_roofline']['stage_ms'])"
 done
done
