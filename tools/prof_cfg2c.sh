python tools/prof_cfg2c.py 256
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2c.csv python tools/prof_cfg2c.py 64 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/launches_cfg2c.csv | head -30
