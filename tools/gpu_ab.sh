# A/B timing of two libocc builds (libocc_A.so vs libocc.so), 3 alternations each
mkdir -p gpurun_out
: > gpurun_out/ab.log
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log >> gpurun_out/ab.log
for i in 1 2 3; do
  echo "A" >> gpurun_out/ab.log; OCC_LIB=$PWD/paper_2408_14050_b200/libocc_A.so timeout 300 python tools/line_stats.py 4 2>&1 | grep "ms per" | tail -1 >> gpurun_out/ab.log
  echo "B" >> gpurun_out/ab.log; timeout 300 python tools/line_stats.py 4 2>&1 | grep "ms per" | tail -1 >> gpurun_out/ab.log
done
