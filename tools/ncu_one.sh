#!/bin/bash
# Full ncu capture of one kernel of a non-graph C2 frame + its hot source lines:
#   bash tools/ncu_one.sh k_small_coop [tag] [launch-skip]
k=$1; tag=${2:-one}; skip=${3:-1}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:$k -s $skip -c 1 -o gpurun_out/${tag} \
    python tools/profile_frame.py C2 3 > gpurun_out/${tag}.log 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/${tag}.ncu-rep
python tools/src_hot.py gpurun_out/${tag}_src.csv 30
