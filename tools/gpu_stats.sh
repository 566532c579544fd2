mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
if grep -q "illegal\|CUDA error\|unspecified launch" gpurun_out/gpu_tests.log; then exit 3; fi
timeout 600 python tools/line_stats.py 4 > gpurun_out/stats.log 2>&1; echo rc=$? >> gpurun_out/stats.log
for cv in 25 75 100; do echo "carveout $cv" >> gpurun_out/stats.log; OCC_LINE_CARVEOUT=$cv timeout 300 python tools/line_stats.py 4 2>&1 | grep "ms per" >> gpurun_out/stats.log; done
if [ -n "$1" ]; then
timeout 300 python tools/prof_family.py $1 4 > gpurun_out/pf.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_line -s 2 -c 1 -o gpurun_out/prof_fam python tools/prof_family.py $1 4 > gpurun_out/ncu_fam.log 2>&1
fi
