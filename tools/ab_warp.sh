for rep in 1 2; do
for lib in old new; do
  L=""; [ $lib = old ] && L="PBP_LIB=paper_1505_04979_b200/_lib/libpbp_old.so"
  for e in 1.0 3.0; do for k in baseline gmatrix csfg; do
    env $L python tools/prof_decode.py --n 1024 --frames 100000 --reps 3 --ebn0 $e --kind $k > gpurun_out/o.txt
    echo "$lib $k $e $(head -1 gpurun_out/o.txt | cut -c14-60) $(tail -1 gpurun_out/o.txt | cut -c1-20)"
  done; done
done; done
