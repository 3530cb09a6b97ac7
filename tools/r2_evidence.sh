# Round-2 evidence on the GPU box: full GPU tests, bench line, reference arm, ncu launch list
# of the bench, full ncu capture of the csfg kernel and per-config rates.
#   bash tools/r2_evidence.sh TAG
set -u
TAG=${1:-r2}
O=gpurun_out; mkdir -p $O
python -m pytest tests -m gpu -q > $O/${TAG}_gputest.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/${TAG}_gputest.log
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_reference_arm.json 2> $O/${TAG}_bench_ref.err; echo "ref rc=$?"
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-gen > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/${TAG}_launch_list.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-gen \
      > $O/${TAG}_ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/prof_decode.py --n 1024 --frames 20000 --reps 1 > /dev/null && \
  ncu --set full --import-source on --clock-control none -k regex:bp_warp_kernel -c 1 \
      -o $O/${TAG}_prof_csfg python tools/prof_decode.py --n 1024 --frames 20000 --reps 1 > $O/${TAG}_ncu_csfg.log 2>&1; echo "ncu csfg rc=$?"
python tools/configs.py > $O/${TAG}_configs.jsonl 2> $O/${TAG}_configs.err; echo "configs rc=$?"
tail -c 600 $O/${TAG}_bench.json
