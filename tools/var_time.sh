# usage: bash tools/var_time.sh v1 v2 ... ("base" = product library): headline mode-A pass times per variant
for v in "$@"; do
  if [ "$v" = base ]; then unset GT_B200_LIB; else export GT_B200_LIB=$PWD/paper_2307_12119_b200/libgreentherm_b200_v$v.so; fi
  python bench.py --steps 40 --no-fp64-line --no-cpu-baseline --no-e2e --no-mode-b --no-cfg2 --no-cfg3 --no-cfg4 2>/dev/null | tail -1 > gpurun_out/var_$v.json
  python -c "import json;d=json.load(open('gpurun_out/var_$v.json'));print('$v',round(d['value']),[round(x,3) for x in d['roofline']['pass_ms_per_step']],'mu1',round(d['per_sample_mu']['value']),d['clocks']['sm_mhz'])"
done
