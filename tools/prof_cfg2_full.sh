# ncu --set full of the config-2 kernels (n = 1024): fp32 mode-B rows / columns, mode-A passes
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:fp_rows<float|fp_cols_d<float|mc_pass[123]w?<float" --launch-skip 2 --launch-count 6 \
    -o gpurun_out/prof_r2_cfg2 -f python tools/prof_cfg2c.py 32 > gpurun_out/prof_r2_cfg2.log 2>&1
tail -1 gpurun_out/prof_r2_cfg2.log
python tools/ncu_summary.py gpurun_out/prof_r2_cfg2.ncu-rep "cfg2" | sed -n 5,30p
