#!/bin/bash
# Per-kernel durations of a few non-graph C2 frames (ncu launch list, cold
# caches, serialised): bash tools/ktimes.sh [tag]
tag=${1:-kt}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/${tag}.csv \
    python tools/profile_frame.py C2 4 > gpurun_out/${tag}.log 2>&1
python tools/launch_table.py gpurun_out/${tag}.csv 2>/dev/null
