# A/B: k_hard batch size (offsets in flight per thread) after the lean scan
# loop: 16 (libocc.so) vs 12 / 20 / 24.
mkdir -p gpurun_out
bash tools/gpu_abenv.sh "b16:OCC_X=1" "b12:OCC_DEFINES=-DHARD_BATCH=12" "b20:OCC_DEFINES=-DHARD_BATCH=20" "b24:OCC_DEFINES=-DHARD_BATCH=24" > gpurun_out/ab5.txt 2>&1
cat gpurun_out/ab5.txt
