# ncu full captures of the n >= 2048 kernels on the current tree (one B200):
#   bash tools/r2_cta_captures.sh TAG
# bp_cta_kernel<12,2> (config 3's kernel, n = 4096) and bp_pair_kernel<13,2> (n = 16384 csfg
# on 2-CTA clusters), 2.5 dB, each after its plain command exited 0
set -u
TAG=${1:-r2}; O=gpurun_out; mkdir -p $O
python tools/prof_decode.py --n 4096 --frames 4440 --reps 1 --ebn0 2.5 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:bp_cta_kernel -c 1 -o $O/${TAG}_prof_cta4096 \
      python tools/prof_decode.py --n 4096 --frames 4440 --reps 1 --ebn0 2.5 > $O/${TAG}_ncu_cta4096.log 2>&1; echo "ncu cta4096 rc=$?"
python tools/prof_decode.py --n 16384 --frames 740 --reps 1 --ebn0 2.5 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:bp_pair_kernel -c 1 -o $O/${TAG}_prof_pair16384 \
      python tools/prof_decode.py --n 16384 --frames 740 --reps 1 --ebn0 2.5 > $O/${TAG}_ncu_pair.log 2>&1; echo "ncu pair rc=$?"
