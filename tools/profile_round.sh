#!/bin/bash
# Round artefacts for profiles/: bench lines (both arms), the ncu launch list
# of the bench command, and one ncu --set full capture of the frame kernels.
# usage (on the GPU box): bash tools/profile_round.sh r1
tag=${1:-r1}
mkdir -p gpurun_out
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err || exit 1
python bench.py --impl reference > gpurun_out/${tag}_bench_reference.json 2> gpurun_out/${tag}_bench_reference.err
# launch list (cold-cache, serialised per-launch times; compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    --profile-frames 0 > gpurun_out/${tag}_ncu_launch.log 2>&1
python tools/launch_table.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches.txt
# full capture of the frame kernels (non-graph path, a few frames)
ncu --set full --metrics lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --import-source on --clock-control none -s 30 -c 40 -o gpurun_out/${tag}_full \
    python tools/profile_frame.py C2 3 > gpurun_out/${tag}_ncu_full.log 2>&1
python tools/ncu_traffic.py gpurun_out/${tag}_full.ncu-rep > gpurun_out/${tag}_ncu_kernels.out
python tools/ncu_summary.py gpurun_out/${tag}_full.ncu-rep > gpurun_out/${tag}_ncu_summary.txt
python tools/bench_configs.py gpurun_out/${tag}_configs.json > gpurun_out/${tag}_configs.log 2>&1
python tools/set_mesh_time.py C3 5 > gpurun_out/${tag}_set_mesh.txt 2>&1
python tools/frame_counters.py C2 4 > gpurun_out/${tag}_counters.txt 2>&1
# whole-frame DRAM traffic in the real cache state (ncu range replay)
bash tools/frame_traffic.sh > /dev/null 2>&1 && cp gpurun_out/traffic.txt gpurun_out/${tag}_frame_traffic.txt
# device-side timeline of graphed frames (FA_TRACE build, tools/lib_trace.so)
if [ -f tools/lib_trace.so ]; then
  FASTATLAS_LIB=tools/lib_trace.so python tools/trace_frame.py C2 16 > gpurun_out/${tag}_trace_c2.txt 2>&1
  FASTATLAS_LIB=tools/lib_trace.so python tools/trace_frame.py C1 16 > gpurun_out/${tag}_trace_c1.txt 2>&1
fi
tail -3 gpurun_out/${tag}_launches.txt
cat gpurun_out/${tag}_ncu_summary.txt | head -40
