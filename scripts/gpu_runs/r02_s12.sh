#!/bin/bash
# round 2 (session 3): the whole GPU suite, the default bench line (config 2 + configs 1/3/4/5),
# the config-1 bench line, and an ncu capture of the resident kernel (push boundary)
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > $O/s12_pytest_gpu.log 2>&1
echo "suite rc=$?" >> $O/s12_pytest_gpu.log
tail -n 4 $O/s12_pytest_gpu.log
timeout 900 python bench.py > $O/s12_bench.json 2> $O/s12_bench.err
echo "bench rc=$?" >> $O/s12_bench.err
timeout 300 python bench.py --config 1 --no-extra --no-cpu-baseline > $O/s12_bench_config1.json 2> $O/s12_bench_config1.err
timeout 300 python scripts/prof_one.py --config 1 --variant implicit --T 200 > $O/s12_prof1.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:resident_kernel -s 1 -c 1 -o $O/s12_resident_c1 -f python scripts/prof_one.py --config 1 --variant implicit --T 200 > $O/s12_ncu_res.log 2>&1
python scripts/ncu_summary.py $O/s12_resident_c1.ncu-rep 30 > $O/s12_resident_c1_summary.txt 2>&1
ncu -i $O/s12_resident_c1.ncu-rep --page source --csv --print-source sass > $O/s12_resident_sass.csv 2>/dev/null
python scripts/sass_stalls.py $O/s12_resident_sass.csv > $O/s12_resident_sass_stalls.txt 2>&1
rm -f $O/*.ncu-rep $O/s12_resident_sass.csv
tail -n 2 $O/s12_bench.err
python - <<'PY'
import json
d=json.load(open("gpurun_out/s12_bench.json"))
print("headline", d["value"], d["roofline"]["frac"], d["e2e"]["value"] if d.get("e2e") else None, d["clocks"])
for k,v in d.get("configs",{}).items(): print(k, v["value"], v["roofline"]["bound"], v["roofline"]["frac"], v["config"].get("variant"), v.get("clocks"))
for a in d.get("alt_variants",[]): print("alt", a["variant"], a["value"], a["roofline"]["frac"])
d=json.load(open("gpurun_out/s12_bench_config1.json"))
print("config1", d["value"], d["roofline"], d["e2e"]["value"] if d.get("e2e") else None)
PY
