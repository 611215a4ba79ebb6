#!/bin/bash
# GPU-box script for a round's committed profiles: the bench launch list (the
# contract's --metrics gpu__time_duration.sum --clock-control none pass over
# the SAME bench command, short), and --set full captures of one frame's conv
# kernels, map kernels and the standalone interleave kernels.  Each ncu run is
# preceded by the same command without ncu (it must exit 0 first).
set -x
mkdir -p gpurun_out
TAG=${TAG:-r2}
BENCH="bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-froxelize --no-train --no-config3 --no-config4"
timeout 600 python $BENCH > gpurun_out/${TAG}_bench_short.json 2> gpurun_out/${TAG}_bench_short.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
      python $BENCH > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 300 python tools/prof_frame.py 1 > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"spconv_(tc|halo)_kernel" -c 15 \
      -o gpurun_out/conv_full_${TAG} python tools/prof_frame.py 1 > gpurun_out/ncu_conv.log 2>&1
ncu --set full --clock-control none -k regex:"l0_flags|compact_levels|tables_kernel|rowbits_grid" -c 7 \
    -o gpurun_out/maps_full_${TAG} python tools/prof_frame.py 1 > gpurun_out/ncu_maps.log 2>&1
timeout 300 python tools/interleave_prof.py > gpurun_out/il_plain.log 2>&1 && \
  ncu --set full --clock-control none -k regex:"il_|deil_" -c 8 -o gpurun_out/il_full_${TAG} \
      python tools/interleave_prof.py > gpurun_out/ncu_il.log 2>&1
tail -2 gpurun_out/*.log
