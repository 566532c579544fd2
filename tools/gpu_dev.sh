# usage: bash tools/gpu_dev.sh [ncu-kernel-regex]
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
if grep -q "illegal\|CUDA error\|unspecified launch" gpurun_out/gpu_tests.log; then echo "CUDA fault: skipping bench/ncu"; exit 3; fi
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-budget 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -n "$1" ]; then
  timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu --frames 32 > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s 8 -c 1 -o gpurun_out/prof_dev python bench.py --steps 1 --warmup 3 --no-cpu --frames 32 > gpurun_out/ncu_full.log 2>&1
fi
echo done
