#!/bin/bash
# DRAM / L2 traffic of one C2 frame in the real cache state (ncu range replay
# around the 5th non-graph frame of one engine, tools/frame_traffic.py):
#   bash tools/frame_traffic.sh            -> gpurun_out/traffic.txt
#   bash tools/frame_traffic.sh stages     (also each stage's range; dirty L2
#       lines of earlier stages are written back inside later ranges, so the
#       per-stage split is indicative only)
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
run() { ncu --replay-mode range --cache-control none --clock-control none --metrics $M \
            python tools/frame_traffic.py C2 nograph 2>&1 | grep -E "dram__bytes|lts__t_bytes" | awk '{print $1, $2, $3}' | tr '\n' ' '; echo; }
names=("project+clear" "depth pass" "visibility pass" "visible compaction" "union-find" "chart roots" "bounds+dims" "order" "pack+select" "uv")
{
  echo "frame: $(run)"
  if [ "$1" = stages ]; then
    for k in 0 1 2 3 4 5 6 7 8 9; do
      echo "stage $k ${names[$k]}: $(FASTATLAS_PROFILE_STAGE=$k run)"
    done
  fi
} > gpurun_out/traffic.txt
cat gpurun_out/traffic.txt
