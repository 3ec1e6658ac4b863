#!/bin/bash
python tools/kbench.py --layers 8 --steps 3 > gpurun_out/kb_auto.json 2>&1
python tools/kbench.py --layers 8 --steps 3 --tune recall_mode=1 > gpurun_out/kb_zc.json 2>&1
python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
python - <<'PY'
import json
for f in ["gpurun_out/kb_auto.json", "gpurun_out/kb_zc.json"]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, open(f).read()[-2000:]); continue
    for k, r in d.items():
        print(f, k, "step %.3f ms, per layer %.1f us" % (r["step_ms"], 1e3 * r["per_layer_ms"]),
              {kk: round(r[kk]["mean_us"], 1) for kk in ("score", "select", "recall")})
PY
