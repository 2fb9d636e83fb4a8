set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_mc_gpu.py -x -q 2>&1 | tail -15
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-mode-b --no-cfg2 --no-cfg3 --no-cfg4 --no-e2e > gpurun_out/b_mf.json 2> gpurun_out/b_mf.err
tail -3 gpurun_out/b_mf.err
python -c "import json;d=json.load(open('gpurun_out/b_mf.json'));print(d['value'],d['ms_per_step'],d['roofline']['pass_ms_per_step'],d['per_sample_mu'],d['fp64_residual_check'],d['clocks'])"
