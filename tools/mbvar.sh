# usage: bash tools/mbvar.sh v1 v2 ...  ("base" = product library): mode-A value and mode-B sub-benchmark per variant
for v in "$@"; do
  if [ "$v" = base ]; then unset GT_B200_LIB; else export GT_B200_LIB=$PWD/paper_2307_12119_b200/libgreentherm_b200_v$v.so; fi
  python bench.py --no-e2e --no-cfg2 --no-cfg3 --no-cfg4 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/mb_$v.json
  python -c "import json;d=json.load(open('gpurun_out/mb_$v.json'));m=d['mode_b']['linear_law'];print('$v',round(d['value']),round(m['value']),m['ms_per_step'],m['mean_iterations'])"
done
