run() { OCC_LINE_WARPS=$1 OCC_LINE_CARVEOUT=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs --no-small 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nw $1 cv $2', round(d['ms_per_step'],2))"; }
run 2 100; run 3 100; run 4 100; run 1 100
