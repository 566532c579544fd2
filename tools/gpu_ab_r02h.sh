# A/B: k_hard entries carrying v_p and an fp32 fixed point + block-maximum
# gating of long searches (libocc.so) vs the gate compiled out (HARD_GATE
# huge) vs the previous commit's library (libocc_head.so): C5 step and the
# h sweep (the gate targets h >= 96).  Outputs in gpurun_out/.
mkdir -p gpurun_out
L=$PWD/paper_2408_14050_b200
timeout 1200 python -m pytest tests/test_gpu_hrange.py tests/test_gpu_queue.py tests/test_gpu_parity.py tests/test_gpu_extremes.py tests/test_gpu_knights.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab2_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab2_tests.log
if grep -q "illegal\|unspecified launch" gpurun_out/ab2_tests.log; then echo "CUDA fault: stop"; exit 3; fi
bash tools/gpu_abenv.sh "head:OCC_LIB=$L/libocc_head.so" "new:OCC_X=1" "gateoff:OCC_DEFINES=-DHARD_GATE=1073741824" > gpurun_out/ab2.txt 2>&1
for v in "head:OCC_LIB=$L/libocc_head.so" "new:OCC_X=1" "gateoff:OCC_DEFINES=-DHARD_GATE=1073741824"; do
  echo "${v%%:*}" >> gpurun_out/ab2_h.txt
  env ${v#*:} timeout 600 python tools/h_sweep.py >> gpurun_out/ab2_h.txt 2>&1
done
tail -3 gpurun_out/ab2_tests.log; cat gpurun_out/ab2.txt
