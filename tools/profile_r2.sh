# Round-2 profiling of the headline (run on the GPU box from the repo root):
#  1. launch list of the bench's timed kernels (serialised, cold cache: compare shares)
#  2. ncu --set full of one 1024-pair launch of each fp32 mode-A pass (gs.mu semantics)
set -x
python bench.py --steps 20 --warmup 3 --no-e2e --no-mode-b --no-cfg2 --no-cfg3 --no-cfg4 --no-cpu-baseline \
    --no-fp64-line > gpurun_out/bench_r2prof.json 2> gpurun_out/bench_r2prof.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-mode-b --no-cfg2 --no-cfg3 --no-cfg4 --no-cpu-baseline \
    --no-fp64-line > gpurun_out/ncu_launch_r2.log 2>&1
ncu --set full --import-source on --clock-control none --cache-control none \
    --kernel-name-base demangled -k "regex:mc_pass[0-9]w?<float" --launch-skip 3 --launch-count 3 \
    -o gpurun_out/prof_r2_modeA -f python tools/prof_mc.py 1024 1024 0 0 0 > gpurun_out/prof_r2_modeA.log 2>&1
tail -2 gpurun_out/prof_r2_modeA.log
