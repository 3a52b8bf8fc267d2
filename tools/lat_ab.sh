# same-box latency A/B of the single-frame path variants (tools/latency_probe.py), alternated
set -u
for rep in 1 2; do
for cfg in "GPUFV_FIN_FUSED=0" "GPUFV_FIN_FUSED=1" ; do
  for n in 5000 8000 17714; do
    echo -n "$cfg N=$n: "; env $cfg PROBE_N=$n timeout 120 python tools/latency_probe.py 2>&1 | tail -1
  done
done
done
