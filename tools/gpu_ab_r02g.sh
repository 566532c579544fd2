# Round-2 (last session) A/B pass: k_hard entries carrying v_p and the fixed
# point (libocc.so) vs the previous commit's library (libocc_head.so), the
# k_hard register cap, chunk alternation; single-frame latency vs the sweep's
# fill target.  Outputs in gpurun_out/.
mkdir -p gpurun_out
L=$PWD/paper_2408_14050_b200
timeout 900 python -m pytest tests/test_gpu_queue.py tests/test_gpu_parity.py tests/test_gpu_extremes.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_tests.log
if grep -q "illegal\|unspecified launch" gpurun_out/ab_tests.log; then echo "CUDA fault: stop"; exit 3; fi
bash tools/gpu_abenv.sh "head:OCC_LIB=$L/libocc_head.so" "new:OCC_X=1" "minb3:OCC_DEFINES=-DHARD_MINB=3" "alt:OCC_ALT=1" > gpurun_out/ab.txt 2>&1
for f in 16 32 64; do echo -n "fill $f: " >> gpurun_out/small.txt; OCC_SWEEP_FILL=$f timeout 120 python tools/small_time.py 3 >> gpurun_out/small.txt 2>&1; OCC_SWEEP_FILL=$f timeout 120 python tools/small_time.py 2 >> gpurun_out/small.txt 2>&1; done
cat gpurun_out/ab.txt gpurun_out/small.txt
