# A/B of the k_cand pre-pass (OCC_LINE_CAND=0 disables it)
for i in 1 2; do for v in 1 0; do
  echo -n "cand=$v: "; OCC_LINE_CAND=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs --no-small 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['roofline']['kernels_ms_per_step']['line'],2), round(d['e2e']['ms_per_step'],2), round(d['device_bits']['ms_per_step'],2))"
done; done
