# Round-2 closing run on one B200 (from the repo root): smoke, GPU tests, the full default
# bench, the reference arm, and the launch list of the bench's timed kernels.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python -m pytest tests -m gpu -q > gpurun_out/gputest_final.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/gputest_final.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-mode-b --no-cfg2 --no-cfg3 --no-cfg4 --no-cpu-baseline \
    --no-fp64-line > gpurun_out/ncu_launch_final.log 2>&1; echo ncu rc=$?
