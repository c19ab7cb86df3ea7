#!/bin/bash
# short bench line (no extras) + x3 variant, for doc numbers after a change
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=${1:-qb}
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python - "$TAG" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/{sys.argv[1]}_bench.json").read().strip().splitlines()[-1])
print("value", round(d["value"]), "e2e", round(d["e2e"]["value"]), "frac", round(d["roofline"]["frac"], 3), "mhz", d["clocks"]["sm_mhz"], "lat", d["latency_b1"]["device_ms"]["p50"])
for k, v in (d.get("precision_variants") or {}).items():
    print(k, round(v["value"]), v["roofline"]["kernel"], round(v["roofline"]["frac"], 3), v["roofline"].get("issued_frac"))
ex = d.get("extra_configs") or {}
for r in ex.get("cfg5_sweep", []):
    if r.get("precision") == "bf16x3" and "slots_per_s" in r:
        print("x3 sweep", r["batch"], round(r["slots_per_s"]))
for k in ("cfg1_bf16x3_b64", "cfg3_bf16x3_b64"):
    if k in ex and "slots_per_s" in ex[k]:
        print(k, round(ex[k]["slots_per_s"]), round(ex[k]["ms_per_step_median"], 3))
PY
