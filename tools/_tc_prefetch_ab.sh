# A/B of the tc_gemm3 L2 prefetch distance (NMFB_TC_PREFETCH) on the C2 bench
for pd in 0 6 8 12 16 0; do
  NMFB_TC_PREFETCH=$pd timeout 300 python bench.py --no-e2e --no-cpu --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split(chr(10))[-1]); print('pd=$pd', round(d['ms_per_step'],4), round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],3))"
done
