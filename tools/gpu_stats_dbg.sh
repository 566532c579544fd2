# event statistics with a debug build of libocc (OCC_LINE_STATS)
mkdir -p gpurun_out
OCC_LINE_STATS=1 python -c "from paper_2408_14050_b200 import build; build.build(force=True)" > gpurun_out/dbg_build.log 2>&1
timeout 600 python tools/line_stats.py 4 > gpurun_out/stats_dbg.log 2>&1
