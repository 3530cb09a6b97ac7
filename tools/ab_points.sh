# per-point timings of the n = 1024 decoders (10^5 frames of config 2 per point),
# for each library build listed in LIBS (default: the in-tree libpbp.so)
set -u
L=$PWD/paper_1505_04979_b200/_lib
for e in ${EBN0:-1.0 3.0 4.0}; do for k in ${KINDS:-csfg}; do
  for lib in ${LIBS:-libpbp.so}; do
    echo "$lib $k $e $(PBP_LIB=$L/$lib timeout 120 python tools/prof_decode.py --n 1024 --frames 100000 --reps 3 --ebn0 $e --kind $k | tail -1)"
  done
done; done
