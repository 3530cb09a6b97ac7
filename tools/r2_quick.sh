# quick GPU check: parity tests of the warp kernel, then per-point timings (n = 1024, 10^5 frames)
set -u
O=gpurun_out; mkdir -p $O
T=${1:-r2x}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > $O/${T}_parity.log 2>&1; echo "parity rc=$?"; tail -3 $O/${T}_parity.log
for k in csfg gmatrix baseline; do for e in 1.0 3.0 4.0; do
  echo "$k $e $(timeout 120 python tools/prof_decode.py --n 1024 --frames 100000 --reps 3 --ebn0 $e --kind $k | tail -1)"
done; done > $O/${T}_points.txt 2>&1
cat $O/${T}_points.txt
