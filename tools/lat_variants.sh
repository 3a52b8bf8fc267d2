set -u
for rep in 1 2 3; do for v in base wchunk; do cp abv/lib_$v.so paper_1604_03498_b200/libgpufv.so; for n in 5000 17714; do echo -n "$v N=$n: "; PROBE_N=$n timeout 120 python tools/latency_probe.py 2>&1 | tail -1; done; done; done
