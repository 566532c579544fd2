# A/B: K0 (k_words) with interior y-blocks specialised (no per-row range
# predicates; libocc.so) vs the previous commit's library (libocc_head.so).
mkdir -p gpurun_out
L=$PWD/paper_2408_14050_b200
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extremes.py tests/test_gpu_hrange.py tests/test_gpu_queue.py tests/test_gpu_packed.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab3_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab3_tests.log
if grep -q "illegal\|unspecified launch" gpurun_out/ab3_tests.log; then echo "CUDA fault: stop"; exit 3; fi
bash tools/gpu_abenv.sh "head:OCC_LIB=$L/libocc_head.so" "interior:OCC_X=1" > gpurun_out/ab3.txt 2>&1
bash tools/gpu_abenv.sh "head:OCC_LIB=$L/libocc_head.so" "interior:OCC_X=1" >> gpurun_out/ab3.txt 2>&1
tail -3 gpurun_out/ab3_tests.log; cat gpurun_out/ab3.txt
