#!/bin/bash
python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for args in "--tune score_ctas_per_sm=0" "--tune score_ctas_per_sm=2" "--tune score_ctas_per_sm=3" "--tune score_ctas_per_sm=2 --tune score_stages=6" "--tune score_ctas_per_sm=1 --tune score_stages=8"; do
  python tools/timeline.py --layers 8 $args 2>&1 | tail -1 | sed "s/^/$args: /"
  python tools/kbench.py --layers 8 --steps 3 $args > /tmp/kb.json 2>&1
  python - "$args" <<'PY'
import json, sys
d = json.load(open("/tmp/kb.json"))
for k, r in d.items():
    print(sys.argv[1], k, "per layer %.1f us" % (1e3 * r["per_layer_ms"]),
          {kk: round(r[kk]["mean_us"], 1) for kk in ("score", "select", "recall")})
PY
done
