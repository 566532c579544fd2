# A/B/C over libocc variants named on the command line (paper_2408_14050_b200/libocc_<name>.so; "base" = libocc.so)
for i in 1 2; do
  for L in "$@"; do
    if [ $L = base ]; then LIB=$PWD/paper_2408_14050_b200/libocc.so; else LIB=$PWD/paper_2408_14050_b200/libocc_$L.so; fi
    echo -n "$L: "; OCC_LIB=$LIB timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs --no-small 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['roofline']['kernels_ms_per_step']['line'],2), round(d['e2e']['ms_per_step'],2))"
  done
done
