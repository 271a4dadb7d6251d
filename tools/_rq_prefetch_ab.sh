# A/B of the residual_i8 L2 prefetch distance (NMFB_RQ_PREFETCH) on the C2 bench
for pd in 0 4 8 0; do
  NMFB_RQ_PREFETCH=$pd timeout 300 python bench.py --no-e2e --no-cpu --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print('pd=$pd', round(d['ms_per_step'],4), round(d['kernels']['nmfb_residual_i8']['avg_ms'],4))"
done
