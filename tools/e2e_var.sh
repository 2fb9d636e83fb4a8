# usage: bash tools/e2e_var.sh v1 v2 ... ("base" = product library): end-to-end host-API rate per variant
for v in "$@"; do
  if [ "$v" = base ]; then unset GT_B200_LIB; else export GT_B200_LIB=$PWD/paper_2307_12119_b200/libgreentherm_b200_v$v.so; fi
  python bench.py --steps 30 --no-cpu-baseline --no-mode-b --no-cfg2 --no-cfg3 --no-cfg4 --no-fp64-line 2>/dev/null | tail -1 > gpurun_out/e2e_$v.json
  python -c "import json;d=json.load(open('gpurun_out/e2e_$v.json'));e=d['e2e'];print('$v',round(e['value']),round(e['ms_per_step'],2),round(e['with_host_variation_maps']['value']))"
done
