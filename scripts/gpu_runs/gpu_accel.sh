timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "accelerated" 2>&1 | tail -15
python - <<'PY'
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, paper_2006_07057_b200 as L
from test_gpu_parity import _accel_pair
for c, n, m, T in [(1, 500, 500, 60), (2, 4099, 3907, 60), (3, 3001, 2999, 40)]:
    gpu, ref, _ = _accel_pair(L, c, n, m, T)
    g = ref["grad_norms"]; rel = np.abs(g[:, 0] - g[:, 1]) / (g[:, 0] + g[:, 1])
    diff = np.nonzero(gpu["blocks"] != ref["blocks"])[0]
    print(c, "first block diff", diff[:3], "min rel margin before", rel[:diff[0]+1].min() if diff.size else rel.min(),
          "F maxrel", np.max(np.abs(gpu["F_trace"] - ref["F_trace"]) / np.abs(ref["F_trace"])))
PY
