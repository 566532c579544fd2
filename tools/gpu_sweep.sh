mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log > gpurun_out/stats.log
for nw in 1 2 4; do for cv in 40 60 100; do echo "warps $nw carve $cv" >> gpurun_out/stats.log; OCC_LINE_WARPS=$nw OCC_LINE_CARVEOUT=$cv timeout 300 python tools/line_stats.py 4 2>&1 | grep "ms per" | tail -1 >> gpurun_out/stats.log; done; done
