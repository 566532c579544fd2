# k_line launch-shape sweep on the bench workload (frame-major order, 2 GiB chunks)
for nw in 1 2 4; do for cv in 40 60 80 100; do
  echo -n "warps $nw carve $cv: "; OCC_LINE_WARPS=$nw OCC_LINE_CARVEOUT=$cv timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['roofline']['kernels_ms_per_step']['line'],2))"
done; done
