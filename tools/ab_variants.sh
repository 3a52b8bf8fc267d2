#!/bin/bash
# A/B library variants built into variants/ (same box, alternating), e.g.
#   bash tools/ab_variants.sh "old new" 3            C4 throughput (the headline)
#   WL=c5 bash tools/ab_variants.sh "old new" 3      C5 dims on a 2M-row set (wide kernel)
#   WL=embed bash tools/ab_variants.sh "old new" 3   raw SIFT -> FV at D = 82 (wide kernel, K = 256)
#   WL=em bash tools/ab_variants.sh "old new" 3      one EM iteration (narrow kernel, exact mode)
vs=${1:-"old"}; reps=${2:-3}; wl=${WL:-c4}
case $wl in
  c4) args="--steps 20 --no-latency --cpu-seconds 0 --e2e-steps 0 --no-legs --score-steps 0";;
  c5) args="--workload c5 --c5-n 2000000 --steps 10 --cpu-seconds 0";;
  embed) args="--workload embed --frames 512 --steps 10 --cpu-seconds 0";;
  em) args="--workload em --steps 10 --cpu-seconds 0";;
esac
for rep in $(seq $reps); do
for v in $vs; do
  cp ${VDIR:-variants}/lib_$v.so paper_1604_03498_b200/libgpufv.so
  a=$(timeout 300 python bench.py $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']/1e9,4), round(d['ms_per_step'],3), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))")
  echo "$rep $v $wl: $a"
done; done
