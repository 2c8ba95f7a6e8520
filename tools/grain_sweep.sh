#!/bin/bash
# CTA-grain sweep for the config-2 projector launches (tools/grain_timing.py);
# run under gpurun from the repo root, output in gpurun_out/grain.log
set -u
O=gpurun_out/grain.log
: > $O
for sp in 1 2 3 4; do PT_GATHER_SPLIT=$sp timeout 300 python tools/grain_timing.py >> $O 2>&1; done
for g in 2 8 12 16 24 32; do PT_FWD_GROUPS=$g timeout 300 python tools/grain_timing.py >> $O 2>&1; done
timeout 300 python tools/grain_timing.py >> $O 2>&1
cat $O
