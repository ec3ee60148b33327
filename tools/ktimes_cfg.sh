#!/bin/bash
# Per-kernel durations of a few non-graph frames of a config: bash tools/ktimes_cfg.sh C1 tag
cfg=${1:-C1}; tag=${2:-ktc}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/${tag}.csv \
    python tools/profile_frame.py $cfg 4 > gpurun_out/${tag}.log 2>&1
python tools/launch_table.py gpurun_out/${tag}.csv 2>/dev/null
