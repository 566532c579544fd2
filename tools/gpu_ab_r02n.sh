# A/B: k_sweep's diagonal uint8 stores by pointer steps and a shifted word
# (-DSWEEP_STORE_LEAN=1) vs libocc.so.
mkdir -p gpurun_out
OCC_DEFINES=-DSWEEP_STORE_LEAN=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hrange.py tests/test_gpu_knights.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab7_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab7_tests.log
if grep -q "illegal\|unspecified launch" gpurun_out/ab7_tests.log; then echo "CUDA fault: stop"; exit 3; fi
bash tools/gpu_abenv.sh "base:OCC_X=1" "storelean:OCC_DEFINES=-DSWEEP_STORE_LEAN=1" > gpurun_out/ab7.txt 2>&1
bash tools/gpu_abenv.sh "base:OCC_X=1" "storelean:OCC_DEFINES=-DSWEEP_STORE_LEAN=1" >> gpurun_out/ab7.txt 2>&1
tail -3 gpurun_out/ab7_tests.log; cat gpurun_out/ab7.txt
