#!/bin/bash
# per-kernel warm-cache launch table (ncu, no cache flush) of a few C2 frames
# through the non-graph path; shares are meaningful, absolutes are serialised
# usage: bash tools/lt.sh [tag]
tag=${1:-warm}
python tools/profile_frame.py C2 2 > /dev/null || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/lt_$tag.csv python tools/profile_frame.py C2 6 > gpurun_out/lt_$tag.log 2>&1
python tools/launch_table.py gpurun_out/lt_$tag.csv
