#!/bin/bash
# round 2, final session: full ncu capture of the d = 16 FFMA feature map (config 3)
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python scripts/time_features.py 3 > $O/r02z_c3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:feature_map_direct -s 6 -c 1 -o $O/r02z_fmap_c3 -f python scripts/time_features.py 3 > $O/r02z_ncu.log 2>&1
cat $O/r02z_c3.log; tail -3 $O/r02z_ncu.log
