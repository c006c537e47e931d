#!/bin/bash
# round 2, call o: full capture of the K3 feature map (3xFP16), summarised on the box
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:feature_map_kernel -s 2 -c 1 -o /tmp/r02o_ftc -f python scripts/time_features.py > $O/r02o_ncu_ftc.log 2>&1
echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/r02o_ftc.ncu-rep 30 > $O/r02o_ftc_summary.txt 2>&1
ncu -i /tmp/r02o_ftc.ncu-rep --page raw --csv > $O/r02o_ftc_raw.csv 2>/dev/null
