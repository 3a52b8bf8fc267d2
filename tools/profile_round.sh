#!/usr/bin/env bash
# Run on the GPU box (gpurun): launch list of the bench command + ncu --set full captures of the
# stats kernel on the full C4 workload, of k_finalize (C4), of the wide stats kernel (C5 shape,
# 2M rows) and of k_embed (raw -> D=82 embedding, 256 frames).  Outputs land in gpurun_out/ (scratch); tools/ncu_summary.py turns them into the
# committed profiles/ summaries.
set -u
TAG=${1:-r01}
python __graft_entry__.py
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_gpu.txt
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-latency --cpu-seconds 0 \
  > gpurun_out/${TAG}_launches.log 2>&1
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:k_stats -s 3 -c 1 \
  -o gpurun_out/${TAG}_kstats python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-latency --cpu-seconds 0 \
  > gpurun_out/${TAG}_kstats.log 2>&1
tail -2 gpurun_out/${TAG}_kstats.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_finalize -s 3 -c 1 \
  -o gpurun_out/${TAG}_finalize python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-latency --cpu-seconds 0 \
  > gpurun_out/${TAG}_finalize.log 2>&1
tail -1 gpurun_out/${TAG}_finalize.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_stats_w -s 3 -c 1 \
  -o gpurun_out/${TAG}_kstats_w python bench.py --workload c5 --c5-n 2000000 --steps 1 --warmup 3 --e2e-steps 0 \
  > gpurun_out/${TAG}_kstats_w.log 2>&1
tail -1 gpurun_out/${TAG}_kstats_w.log
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_embed -s 3 -c 1 \
  -o gpurun_out/${TAG}_embed python bench.py --workload embed --frames 256 --steps 1 --warmup 3 \
  > gpurun_out/${TAG}_embed.log 2>&1
tail -1 gpurun_out/${TAG}_embed.log
# single-frame latency path (C2 shape): per-kernel durations of the prepared encode (serialised)
PROBE_REPS=3 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv \
  --log-file gpurun_out/${TAG}_latency_launches.csv python tools/latency_probe.py > gpurun_out/${TAG}_latency.log 2>&1
python tools/latency_probe.py >> gpurun_out/${TAG}_latency.log 2>&1
tail -1 gpurun_out/${TAG}_latency.log
