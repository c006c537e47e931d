#!/bin/bash
# round 2: compute-sanitizer, ONE tool per gpurun call (B200_PROFILING.md): bash r02_san.sh <tool>
# every case of scripts/sanitize_case.py first runs plainly (exit 0) — then under the tool
cd $GRAFT_REPO_ROOT
O=gpurun_out
tool=${1:-racecheck}
timeout 300 python scripts/sanitize_case.py > $O/r02_san_plain.log 2>&1 || { echo "plain run failed"; tail $O/r02_san_plain.log; exit 1; }
for c in c1_stream c1_implicit c2_stream c2_implicit tol_stream tol_implicit batched emul_stream emul_implicit; do
  echo "== $c" >> $O/r02_san_$tool.log
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py $c >> $O/r02_san_$tool.log 2>&1
  echo "rc=$?" >> $O/r02_san_$tool.log
done
grep -E "^==|rc=|ERROR SUMMARY|RACECHECK SUMMARY|hazard|Error" $O/r02_san_$tool.log | head -80
