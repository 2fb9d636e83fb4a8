# config-2 variants: correctness of the product library, then the combined solve per variant
set -x
timeout 900 python -m pytest tests/test_config2_gpu.py tests/test_fixed_point_gpu.py tests/test_large_gpu.py -x -q > gpurun_out/t_c2.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/t_c2.log
bash tools/c2c_time.sh base kpow nghs ub2 base > gpurun_out/c2var.log 2>&1
cat gpurun_out/c2var.log
