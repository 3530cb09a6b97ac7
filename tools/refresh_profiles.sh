#!/usr/bin/env bash
# Regenerate the measured evidence under gpurun_out/ (run on the GPU box):
#   bash tools/refresh_profiles.sh TAG
# bench line (+ reference arm), ncu launch list of the bench, one full ncu
# capture of the csfg and the baseline decoder kernels, and the section split
# (tools/prof_decode.py) - each ncu pass only after its plain command exited 0.
set -u
TAG=${1:-r1}
O=gpurun_out
mkdir -p $O
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err || exit 1
python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_reference_arm.json 2> $O/${TAG}_bench_ref.err || exit 1
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/${TAG}_launch_list.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
      > $O/${TAG}_ncu_launch.log 2>&1
python tools/prof_decode.py --n 1024 --frames 20000 --reps 1 > /dev/null && \
  ncu --set full --import-source on --clock-control none -k regex:bp_warp_kernel -c 1 \
      -o $O/${TAG}_prof_csfg python tools/prof_decode.py --n 1024 --frames 20000 --reps 1 > $O/${TAG}_ncu_csfg.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bp_warp_kernel -c 1 \
    -o $O/${TAG}_prof_base python tools/prof_decode.py --n 1024 --frames 20000 --reps 1 --kind baseline \
    > $O/${TAG}_ncu_base.log 2>&1
ncu --set full --clock-control none -k regex:bp_warp_kernel -c 1 --metrics dram__bytes_read.sum,dram__bytes_write.sum \
    -o $O/${TAG}_prof_traffic python tools/prof_decode.py --n 1024 --frames 20000 --reps 1 > /dev/null 2>&1
for e in 1.0 2.0 3.0 4.0; do
  echo "== Eb/N0 $e"
  python tools/prof_decode.py --n 1024 --frames 100000 --reps 2 --ebn0 $e | tail -1
done > $O/${TAG}_points.txt
tail -1 $O/${TAG}_bench.json
