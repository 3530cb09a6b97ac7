# decode throughput of the CTA kernel at n = 2048..16384, 2.5 dB (tools/prof_decode.py)
NS=${NS:-"2048 4096 8192 16384"}; KS=${KS:-"csfg gmatrix baseline"}
for n in $NS; do
  f=$((20000*1024/n)); [ $f -lt 2000 ] && f=2000
  for k in $KS; do
    echo "n=$n $k: $(python tools/prof_decode.py --n $n --kind $k --ebn0 2.5 --frames $f --reps 3 2>&1 | tail -1)"
  done
done
