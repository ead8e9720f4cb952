#!/bin/bash
# C4 KV-pressure sweep on one B200 (scaled to one GPU): 8B shape,
# 32k-token initial contexts, the 4 default decode modules, concurrency caps
# swept, both serving modes, decode-side residency + staged handoff (copy).
mkdir -p gpurun_out/kvp
timeout 3000 python tools/run_agents.py --shape 8b --pattern react --initial-prompt-len 32768 \
  --max-context 35200 --rate 0.5 --duration 20 --sweep max_concurrent_sessions --values 1,2,4,8 \
  --rows 8 --pool-pages 4096 --handoff copy --decode-capacity 3072 --out gpurun_out/kvp \
  > gpurun_out/kvp/run.log 2> gpurun_out/kvp/run.err
echo "kvp rc=$?"; tail -20 gpurun_out/kvp/run.log; tail -5 gpurun_out/kvp/run.err
