mkdir -p gpurun_out
timeout 300 python tools/prof_family.py $1 4 > gpurun_out/pf.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_line -s 2 -c 1 -o gpurun_out/prof_fam python tools/prof_family.py $1 4 > gpurun_out/ncu_fam.log 2>&1
