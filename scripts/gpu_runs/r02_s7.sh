#!/bin/bash
# round 2 (session 3): whole GPU suite and the default bench line with the resident kernel and
# the boundary overlap
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > $O/s7_pytest_gpu.log 2>&1
echo "suite rc=$?" >> $O/s7_pytest_gpu.log
timeout 900 python bench.py > $O/s7_bench.json 2> $O/s7_bench.err
echo "bench rc=$?" >> $O/s7_bench.err
tail -n 5 $O/s7_pytest_gpu.log; tail -n 3 $O/s7_bench.err
python - <<'PY'
import json
d=json.load(open("gpurun_out/s7_bench.json"))
print("headline", d["value"], d["roofline"]["frac"], d["e2e"]["value"] if d.get("e2e") else None, d["clocks"])
for k,v in d.get("configs",{}).items(): print(k, v["value"], v["roofline"]["bound"], v["roofline"]["frac"], v["config"].get("variant"))
for a in d.get("alt_variants",[]): print("alt", a["variant"], a["value"], a["roofline"]["frac"])
PY
