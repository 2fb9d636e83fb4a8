# ncu --set full of the config-3 per-step kernels (n = 512, 64 traces)
ncu --set full --clock-control none --kernel-name-base demangled -k "regex:tr_" --launch-skip 30 --launch-count 3 \
    -o gpurun_out/prof_r2_cfg3 -f python tools/prof_trace.py 512 64 40 > gpurun_out/prof_r2_cfg3.log 2>&1
tail -1 gpurun_out/prof_r2_cfg3.log
python tools/ncu_summary.py gpurun_out/prof_r2_cfg3.ncu-rep "cfg3" | sed -n 5,30p
