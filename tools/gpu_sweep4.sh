run() { OCC_LINE_WARPS=$1 OCC_LINE_CARVEOUT=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nw $1 cv $2', round(d['ms_per_step'],2), round(d['roofline']['kernels_ms_per_step']['line'],2))"; }
for cv in 30 40 45 50; do run 4 $cv; done
for cv in 45 50; do run 3 $cv; done
