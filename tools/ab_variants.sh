#!/bin/bash
# A/B library variants built into variants/ (same box, alternating): C4 throughput per variant.
#   bash tools/ab_variants.sh "old prekc" [reps]
vs=${1:-"old"}; reps=${2:-3}
for rep in $(seq $reps); do
for v in $vs; do
  cp variants/lib_$v.so paper_1604_03498_b200/libgpufv.so
  a=$(timeout 300 python bench.py --steps 20 --no-latency --cpu-seconds 0 --e2e-steps 0 --no-legs --score-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']/1e9,4), round(d['roofline']['kernel_ms'],3), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))")
  echo "$rep $v C4: $a"
done; done
