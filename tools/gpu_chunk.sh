mkdir -p gpurun_out
: > gpurun_out/chunk.log
for mib in 96 160 320 640; do
  echo "chunk MiB $mib" >> gpurun_out/chunk.log
  OCC_CHUNK_MIB=$mib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-fuse 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernels_ms_per_step'])" >> gpurun_out/chunk.log
done
