# A/B of an environment switch on the cfg2 bench: tools/ab_env.sh VAR v1 v2 ...
var=$1; shift
for v in "$@"; do
  env $var=$v timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab_${var}_$v.json 2> gpurun_out/ab_${var}_$v.err
  python - "$var" "$v" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], sys.argv[2], "value", round(d["value"], 1), "serial", round(d.get("value_serial") or 0, 1),
      {k: round(v, 3) for k, v in d.get("phases_ms_per_approx", {}).items()})
PY
done
