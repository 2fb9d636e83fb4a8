# usage: bash tools/c2c_time.sh v1 v2 ... ("base" = product library): config-2 combined solve time per variant
for v in "$@"; do
  if [ "$v" = base ]; then unset GT_B200_LIB; else export GT_B200_LIB=$PWD/paper_2307_12119_b200/libgreentherm_b200_v$v.so; fi
  echo "== $v"; python tools/prof_cfg2c.py 256 2>&1 | tail -2
done
