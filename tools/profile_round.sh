#!/bin/bash
# Profiling pass of one round (run under gpurun on ONE B200; never multi-rank).
#   tools/profile_round.sh TAG
# 1. the kernel-sources hash the captures belong to
# 2. the ncu launch list (gpu__time_duration per launch, cold and serialised)
#    of the bench command
# 3. ncu --set full of the fused tcgen05 fwd/bwd at the bench workload
# 4. ncu --set full of the four split kernels at d = 256 (BASELINE configs[3])
# Summaries are made on the CPU side: tools/ncu_summary.py gpurun_out/prof_TAG.ncu-rep ...
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "from paper_2406_06484_b200.build import sources_sha; print(sources_sha())" \
  > gpurun_out/sha_$TAG.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  -k regex:"tc_|sp_|simt_|rec_fwd|prologue|seg_scan|cp_" \
  --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"tc_(fwd|bwd)_kernel" -s 2 -c 2 -o gpurun_out/prof_$TAG -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-recurrent --no-strong \
  > gpurun_out/prof_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"sp_" -s 4 -c 4 -o gpurun_out/prof_${TAG}_split -f \
  python tools/hd256_time.py 256 > gpurun_out/prof_${TAG}_split.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
ls -la gpurun_out/*$TAG*
