# Round-2 measurement pass (run under gpurun): GPU tests, smoke, the default bench,
# ncu launch lists (all legs; the main step), one `ncu --set full` capture each of
# k_sweep / k_words / k_hard on the main step and of k_shear on C4.  Outputs in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1; nproc >> gpurun_out/smi.txt; lscpu | head -20 >> gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
if grep -q "illegal\|unspecified launch" gpurun_out/gpu_tests.log; then echo "CUDA fault: stop"; exit 3; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
M="--steps 2 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs --no-small --no-e2e"
timeout 600 python bench.py $M > gpurun_out/plain_main.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_main.csv python bench.py $M > gpurun_out/ncu_launch_main.log 2>&1
python tools/launch_shares.py gpurun_out/launches_main.csv > gpurun_out/launch_shares.txt 2>&1
for k in k_sweep k_words k_hard; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python bench.py $M > gpurun_out/ncu_full_$k.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_shear -s 1 -c 1 -o gpurun_out/prof_k_shear python tools/c4_time.py > gpurun_out/ncu_full_k_shear.log 2>&1
timeout 300 python tools/c4_time.py > gpurun_out/c4.txt 2>&1
for k in k_sweep k_words k_hard k_shear; do python tools/ncu_keys.py gpurun_out/prof_$k.ncu-rep >> gpurun_out/ncu_keys.txt 2>&1; done
ncu -i gpurun_out/prof_k_sweep.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ksweep_src.csv 2>/dev/null
python tools/ncu_src_stalls.py gpurun_out/ksweep_src.csv 10 > gpurun_out/ksweep_stalls.txt 2>&1
echo done
