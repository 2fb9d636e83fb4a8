# usage: bash tools/ovl.sh "OVL:CHUNK" ...  -- mode-A bench under GT_MC_OVERLAP / chunk variants
for v in "$@"; do
  o=${v%%:*}; c=${v##*:}
  GT_MC_OVERLAP=$o python bench.py --chunk $c --no-cpu-baseline --no-e2e --no-mode-b --no-cfg2 --no-cfg3 --no-cfg4 2>/dev/null | tail -1 > gpurun_out/ovl_${o}_$c.json
  python -c "import json;d=json.load(open('gpurun_out/ovl_${o}_$c.json'));print('ovl $o chunk $c',round(d['value']),d['failed_pairs'],d['fp64_residual_check']['max_abs_K'],[round(x,3) for x in d['roofline']['pass_ms_per_step']])"
done
