# usage: bash tools/subvar.sh v1 v2 ...  ("base" = product library): mode-B and config-3 sub-benchmarks per variant
for v in "$@"; do
  if [ "$v" = base ]; then unset GT_B200_LIB; else export GT_B200_LIB=$PWD/paper_2307_12119_b200/libgreentherm_b200_v$v.so; fi
  python bench.py --no-e2e --no-cfg2 --no-cfg4 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/sub_$v.json
  python -c "import json;d=json.load(open('gpurun_out/sub_$v.json'));m=d['mode_b']['linear_law'];print('$v',round(d['value']),'modeB',round(m['value']),'cfg3',round(d['cfg3']['value']))"
done
