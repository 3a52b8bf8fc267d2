# same-box latency A/B of the single-frame path settings (tools/latency_probe.py), alternated
# usage: bash tools/lat_ab.sh ["ENV=.. ENV=..;ENV=.."] ["N N .."] [reps]
set -u
IFS=';' read -ra cfgs <<< "${1:-GPUFV_FIN_FUSED=0;GPUFV_FIN_FUSED=1}"
ns=${2:-"5000 8000 17714"}; reps=${3:-2}
for rep in $(seq $reps); do
for cfg in "${cfgs[@]}"; do
  for n in $ns; do
    echo -n "$cfg N=$n: "; env $cfg PROBE_N=$n timeout 120 python tools/latency_probe.py 2>&1 | tail -1
  done
done
done
