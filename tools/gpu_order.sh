# A/B of k_line work order (OCC_LINE_ORDER 0: frames fastest, 1: frame-major), bench-like timing
mkdir -p gpurun_out
for i in 1 2; do for o in 0 1; do
  echo "order=$o"; OCC_LINE_ORDER=$o timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-fuse --nwin 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernels_ms_per_step'])"
done; done
OCC_LINE_ORDER=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_line -s 20 -c 3 python bench.py --steps 2 --warmup 3 --no-cpu --no-fuse --nwin 0 2>&1 | grep -E "dram__|gpu__time" | head -12
