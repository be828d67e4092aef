# L2 evict-first policy on the payload TMA (HM_PAYLOAD_EVICT_FIRST, engine_dev.cuh) on / off:
# C2 64-RHS flux / apply / solve, C2 single-vector flux, and the DRAM bytes of the 64-RHS flux launch
run1() { for r in 1 2; do timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --no-level-form 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('  flux us', round(d['ms_per_step']*1e3,1), 'engine us', round(d['config']['engine_ms']['flux']*1e3,1), 'frac', round(d['roofline']['frac'],4))"; done; }
for d in "HM_PAYLOAD_EVICT_FIRST=1" "HM_PAYLOAD_EVICT_FIRST=0"; do
  HM_BUILD_DEFINES="$d" python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null || exit 1
  echo "== defines: [$d]"
  for r in 1 2; do timeout 600 python scripts/mrhs_bench.py 2>&1 | grep -v "^\[hm\]"; done
  run1
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:engine -c 16 --csv python scripts/mrhs_bench.py 2>/dev/null | grep -E "engine" | python -c "
import sys,csv
rows=list(csv.reader(sys.stdin))
for r in rows:
    if len(r)>14: print('   ', r[4][:24], r[-3], r[-2], r[-1])
" | tail -48
done
python -c "from paper_2305_06891_b200 import build as b; b.build(force=True)" > /dev/null
