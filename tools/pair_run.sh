# A/B of the K1 GEMM kernels (PSK_GEMM_PAIR=0: 1-SM, default: CTA pair) on
# the whole 4k prefill and on the serve bench, alternating to spread clock drift.
for i in 1 2 3; do
  for v in 0 1; do
    echo "PSK_GEMM_PAIR=$v"; PSK_GEMM_PAIR=$v timeout 300 python tools/bench_prefill.py 4096 quick 2>&1 | tail -1
  done
done
for v in 0 1; do
  echo "PSK_GEMM_PAIR=$v bench"; PSK_GEMM_PAIR=$v timeout 600 python bench.py --steps 2 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['prefill'], d['clocks'])"
done
