# A/B over libocc variants (paper_2408_14050_b200/libocc_<name>.so; "base" = libocc.so) on the
# main C5 step: ms/step, per-kernel ms/step and the SHA-256 prefix of the timed masks.
for i in 1 2; do
  for L in "$@"; do
    if [ $L = base ]; then LIB=$PWD/paper_2408_14050_b200/libocc.so; else LIB=$PWD/paper_2408_14050_b200/libocc_$L.so; fi
    echo -n "$L: "; OCC_LIB=$LIB timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs --no-small --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); k=d['roofline']['kernels_ms_per_step']
    print(round(d['ms_per_step'],3), {a: round(b,3) for a,b in k.items()}, d['parity']['sha256_masks'][:12])
except Exception as e: print('FAILED', e)"
  done
done
