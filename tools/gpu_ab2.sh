# A/B: libocc_A.so vs libocc.so on the bench workload (3 alternations), optional env for A
for i in 1 2 3; do
  for L in A B; do
    if [ $L = A ]; then LIB=$PWD/paper_2408_14050_b200/libocc_A.so; else LIB=$PWD/paper_2408_14050_b200/libocc.so; fi
    echo -n "$L: "; OCC_LIB=$LIB timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs --no-small 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['roofline']['kernels_ms_per_step']['line'],2), round(d['e2e']['ms_per_step'],2))"
  done
done
