# launch_bounds(128) build (A) vs launch_bounds(256) build (B): warps per CTA x carve-out
run() { OCC_LIB=$PWD/paper_2408_14050_b200/$1 OCC_LINE_WARPS=$2 OCC_LINE_CARVEOUT=$3 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 nw $2 cv $3', round(d['ms_per_step'],2), round(d['roofline']['kernels_ms_per_step']['line'],2))"; }
for cv in 50 55 60 65 70; do run libocc_A.so 4 $cv; done
for nw in 4 6 8; do for cv in 50 60 70; do run libocc_B.so $nw $cv; done; done
