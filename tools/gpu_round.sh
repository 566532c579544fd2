# Full measurement pass (run under gpurun): GPU tests, smoke, bench, ncu launch list and
# one full ncu capture of the dominant kernel.  Outputs land in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1; nproc >> gpurun_out/smi.txt; lscpu | head -20 >> gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
if grep -q "illegal\|CUDA error\|unspecified launch" gpurun_out/gpu_tests.log; then echo "CUDA fault: stop"; exit 3; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
# the main step only (warm-up + timed steps of the C5 detection): kernel shares of the step
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs --no-small --no-e2e > gpurun_out/plain_main.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_main.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs --no-small --no-e2e > gpurun_out/ncu_launch_main.log 2>&1
M="--steps 2 --warmup 3 --no-cpu --no-fuse --nwin 0 --no-dirs --no-small --no-e2e"
grep -q '"metric"' gpurun_out/plain_main.log && for k in k_sweep k_words k_hard; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python bench.py $M > gpurun_out/ncu_full_$k.log 2>&1
done
echo done
