#!/bin/bash
# depth / latency study with the paper's 3x3 stem / head on every plan precision (round 2, after 3x3 heads)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for prec in bf16 bf16x3; do
  timeout 600 python tools/depth_latency.py 1800000 $prec 200 > gpurun_out/r02b_depth_latency_${prec}_P1.8M.json 2> gpurun_out/r02b_depth_${prec}.err
done
# fp32: timeout 900 python tools/depth_latency.py 1900000 fp32 100 > gpurun_out/r02b_depth_latency_fp32_P1.9M.json 2> gpurun_out/r02b_depth_fp32.err
python - <<'PY'
import json
for f in ("bf16_P1.8M", "bf16x3_P1.8M", "fp32_P1.9M"):
    try:
        d = json.load(open(f"gpurun_out/r02b_depth_latency_{f}.json"))
        print(f, {k: (v["width"], v.get("latency_b1_ms", {}).get("median"), v.get("throughput_b64_slots_per_s")) for k, v in d["nets"].items()}, d.get("latency_reduction_b1"))
    except Exception as e:
        print(f, e)
PY
