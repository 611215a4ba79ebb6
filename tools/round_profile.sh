#!/bin/bash
# GPU-box script: gpu tests, bench, ncu launch list and --set full captures of
# the conv kernels and map kernels of one frame (tools/prof_frame.py).
set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 python tools/prof_frame.py > gpurun_out/prof_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
      python tools/prof_frame.py > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/prof_frame.py > gpurun_out/prof_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"spconv_(tc|halo)_kernel" -c 15 \
      -o gpurun_out/conv_full_${TAG} python tools/prof_frame.py > gpurun_out/ncu_conv.log 2>&1
timeout 300 python tools/prof_frame.py > gpurun_out/prof_plain3.log 2>&1 && \
  ncu --set full --clock-control none -k regex:"l0_flags|compact_levels|tables_kernel|count_kernel|place_kernel|halo_build" -c 6 \
      -o gpurun_out/maps_full_${TAG} python tools/prof_frame.py > gpurun_out/ncu_maps.log 2>&1
tail -3 gpurun_out/*.log
