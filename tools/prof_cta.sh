# ncu evidence for the CTA-per-frame kernel (configs 3 and 4): one full capture per size
#   bash tools/prof_cta.sh TAG
set -u
T=${1:-r2}; O=gpurun_out; mkdir -p $O
for n in 4096 16384; do
  f=$([ $n = 4096 ] && echo 8000 || echo 1480)
  python tools/prof_decode.py --n $n --frames $f --reps 1 --ebn0 2.5 > /dev/null && \
  ncu --set full --import-source on --clock-control none -k regex:bp_cta_kernel -c 1 -o $O/${T}_prof_cta$n \
      python tools/prof_decode.py --n $n --frames $f --reps 1 --ebn0 2.5 > $O/${T}_ncu_cta$n.log 2>&1; echo "ncu cta $n rc=$?"
done
