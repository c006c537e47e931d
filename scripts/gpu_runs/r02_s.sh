#!/bin/bash
# round 2, call s: config 1 (n = m = 500, r = 100) per-pass time vs the CTA group size (tuning
# build: LSK_GPP), both variants
cd $GRAFT_REPO_ROOT
export LSK_LIB_PATH=$GRAFT_REPO_ROOT/scripts/variants/liblsk_tuning.so
for v in implicit stream; do
  for g in 1 2 4 8 16; do
    echo -n "variant $v gpp $g: "; LSK_GPP=$g timeout 120 python scripts/sweep.py --config 1 --variant $v --T 200 --reps 5 2>&1 | tail -1
  done
done
