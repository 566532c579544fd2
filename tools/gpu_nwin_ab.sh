for i in 1 2; do for L in base g64 g128; do
  if [ $L = base ]; then LIB=$PWD/paper_2408_14050_b200/libocc.so; else LIB=$PWD/paper_2408_14050_b200/libocc_$L.so; fi
  echo -n "$L: "; OCC_LIB=$LIB timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-fuse --no-small 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['finite_n']['ms_per_step'],2), round(d['directions']['ms_per_step'],2))"
done; done
