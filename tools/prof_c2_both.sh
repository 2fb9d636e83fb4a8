set -x
bash tools/prof_cfg2c.sh > gpurun_out/c2_launch.txt 2>&1
bash tools/prof_cfg2_full.sh > gpurun_out/c2_full.txt 2>&1
