# c5 (and c4) bench lines for each library variant (PVSPH_LIB=exp/NAME.so; "base" = the in-tree
# build), interleaved twice to expose box noise.  usage: bash scripts/ab_variants.sh "c5 c4" base v1 v2 ...
mkdir -p gpurun_out
CFGS=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then L=""; else L="PVSPH_LIB=$PWD/exp/$v.so"; fi
    for c in $CFGS; do
      env $L timeout 600 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/ab_${v}_${c}_$rep.json 2>/dev/null
      python - $v $c $rep <<'PY'
import json,sys
v,c,r=sys.argv[1:4]
try:
    d=json.loads(open(f"gpurun_out/ab_{v}_{c}_{r}.json").read().strip().splitlines()[-1])
    print(r, v, c, round(d["ms_per_step"],2), {k: round(x,2) for k,x in d["stage_ms"].items()})
except Exception as e: print(r, v, c, "ERR", e)
PY
    done
  done
done
