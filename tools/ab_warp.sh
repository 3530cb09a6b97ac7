# A/B of the warp-resident kernel: a library built from an older bp_warp.cu against the
# current one, every decoder at 1 and 3 dB (n = 1024, 10^5 frames, third repetition).
# Build the old one first, e.g.
#   git show <rev>:paper_1505_04979_b200/csrc/bp_warp.cu > paper_1505_04979_b200/csrc/bp_warp.cu
#   PBP_OBJ_SUBDIR=obj_old PBP_LIB_NAME=libpbp_old.so python paper_1505_04979_b200/build.py
#   git checkout paper_1505_04979_b200/csrc/bp_warp.cu
for rep in 1 2; do
for lib in old new; do
  L=""; [ $lib = old ] && L="PBP_LIB=paper_1505_04979_b200/_lib/libpbp_old.so"
  for e in 1.0 3.0; do for k in baseline gmatrix csfg; do
    env $L python tools/prof_decode.py --n 1024 --frames 100000 --reps 3 --ebn0 $e --kind $k > gpurun_out/o.txt
    echo "$lib $k $e $(head -1 gpurun_out/o.txt | cut -c14-60) $(tail -1 gpurun_out/o.txt | cut -c1-20)"
  done; done
done; done
