# usage: bash tools/c3var.sh v1 v2 ...  ("base" = product library): config-3 sub-benchmark per variant
for v in "$@"; do
  if [ "$v" = base ]; then unset GT_B200_LIB; else export GT_B200_LIB=$PWD/paper_2307_12119_b200/libgreentherm_b200_v$v.so; fi
  python bench.py --steps 3 --no-e2e --no-mode-b --no-cfg2 --no-cfg4 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/c3_$v.json
  python -c "import json;d=json.load(open('gpurun_out/c3_$v.json'));c=d['cfg3'];print('$v',round(c['value']),round(c['ms'],1))"
done
