run() { OCC_LINE_WARPS=$1 OCC_LINE_CARVEOUT=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs --no-small 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nw $1 cv $2', round(d['ms_per_step'],2))"; }
for nw in 2 4; do for cv in 45 60 75 100; do run $nw $cv; done; done
run 1 45; run 3 60
