# same-box single-frame latency A/B of library variants built into ${VDIR:-abv}/lib_<name>.so
set -u
vs=${1:-"base"}; ns=${2:-"5000 17714"}; reps=${3:-3}
for rep in $(seq $reps); do for v in $vs; do cp ${VDIR:-abv}/lib_$v.so paper_1604_03498_b200/libgpufv.so; for n in $ns; do echo -n "$v N=$n: "; PROBE_N=$n timeout 120 python tools/latency_probe.py 2>&1 | tail -1; done; done; done
