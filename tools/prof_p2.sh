# ncu --set full of the mode-A column pass, both closed-form mu semantics (1024-pair launches)
ncu --set full --import-source on --clock-control none -k regex:mc_pass2 --launch-skip 1 --launch-count 3 -o gpurun_out/prof_r2_p2 -f python tools/prof_mc.py 1024 1024 0 both > gpurun_out/prof_r2_p2.log 2>&1
tail -1 gpurun_out/prof_r2_p2.log
python tools/ncu_summary.py gpurun_out/prof_r2_p2.ncu-rep | sed -n 7,30p
