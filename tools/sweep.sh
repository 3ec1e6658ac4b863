#!/bin/bash
# tuning sweep on an 8-layer C2-shaped cache (zero-copy and DMA recall)
for args in "--tune recall_mode=1" "--tune recall_mode=1 --tune score_stages=6" "--tune recall_mode=1 --tune score_stages=8" \
            "--tune recall_mode=1 --tune recall_ctas=148" "--tune recall_mode=1 --tune recall_ctas=64" \
            "--tune recall_mode=1 --tune score_stages=6 --tune recall_ctas=148" "--tune recall_mode=2 --tune score_stages=6"; do
  python tools/kbench.py --layers 8 --steps 3 $args > /tmp/kb.json 2>&1
  python - "$args" <<'PY'
import json, sys
d = json.load(open("/tmp/kb.json"))
for k, r in d.items():
    print(sys.argv[1], k, "per layer %.1f us" % (1e3 * r["per_layer_ms"]),
          {kk: round(r[kk]["mean_us"], 1) for kk in ("score", "select", "recall")})
PY
done
