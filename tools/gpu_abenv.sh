# A/B over environment settings on the main C5 step.  Each argument is
# "label:VAR=val,VAR=val" (OCC_LIB=... selects a library variant); prints
# ms/step, per-kernel ms/step and the SHA-256 prefix of the timed masks.
for i in 1 2; do
  for A in "$@"; do
    label=${A%%:*}; envs=${A#*:}
    echo -n "$label: "
    env $(echo "$envs" | tr ',' ' ') timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs --no-small --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); k=d['roofline']['kernels_ms_per_step']
    print(round(d['ms_per_step'],3), {a: round(b,3) for a,b in k.items()}, d['parity']['sha256_masks'][:12])
except Exception as e: print('FAILED', e)"
  done
done
