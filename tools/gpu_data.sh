# Data pass (run under gpurun): k_sweep event counters (SWEEP_STATS build) and
# a full per-source-line dump of one k_sweep capture on the main C5 step.
mkdir -p gpurun_out
M="--steps 2 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs --no-small --no-e2e"
OCC_DEFINES=-DSWEEP_STATS timeout 300 python tools/sweep_stats.py 8 > gpurun_out/sweep_stats.txt 2>&1
timeout 600 python bench.py $M > gpurun_out/plain_main.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 2 -c 1 -o gpurun_out/prof_k_sweep python bench.py $M > gpurun_out/ncu_full_k_sweep.log 2>&1
ncu -i gpurun_out/prof_k_sweep.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ksweep_src.csv 2>/dev/null
ncu -i gpurun_out/prof_k_sweep.ncu-rep --page source --csv --print-source cuda > gpurun_out/ksweep_cuda.csv 2>/dev/null
ls -la gpurun_out
