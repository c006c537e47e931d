#!/bin/bash
# round 2, final session: feature-map times of the five configurations
cd $GRAFT_REPO_ROOT
timeout 900 python scripts/time_features.py > gpurun_out/r02y_feature_map_times.log 2>&1
echo "rc=$?" >> gpurun_out/r02y_feature_map_times.log
cat gpurun_out/r02y_feature_map_times.log
