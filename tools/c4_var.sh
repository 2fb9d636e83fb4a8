# usage: bash tools/c4_var.sh v1 v2 ... ("base" = product library): config-4 solve time per variant
for v in "$@"; do
  if [ "$v" = base ]; then unset GT_B200_LIB; else export GT_B200_LIB=$PWD/paper_2307_12119_b200/libgreentherm_b200_v$v.so; fi
  echo "$v: $(python bench.py --steps 3 --no-cpu-baseline --no-e2e --no-mode-b --no-cfg2 --no-cfg3 --no-fp64-line 2>/dev/null | python -c 'import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d["cfg4"];print(round(c["ms"],1),"ms",c["iterations"],"it",round(c["ms_per_iteration"],2),"ms/it",round(c["achieved_GBps_model"]),"GB/s")')"
done
