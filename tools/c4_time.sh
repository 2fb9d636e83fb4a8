# usage: bash tools/c4_time.sh v1 v2 ... ("base" = product library): config-4 ms per iteration per variant
for v in "$@"; do
  if [ "$v" = base ]; then unset GT_B200_LIB; else export GT_B200_LIB=$PWD/paper_2307_12119_b200/libgreentherm_b200_v$v.so; fi
  echo "== $v"; python tools/prof_large.py ${C4N:-8192} 2>&1 | grep rep
done
