# A/B of the n = 1024 csfg kernels: PBP_WS=0 (one warp per frame) vs the
# warp-specialised kernel, optionally other library builds (LIBS=..., OLDLIBS=... run with PBP_WS=0)
set -u
L=$PWD/paper_1505_04979_b200/_lib
for e in ${EBN0:-1.0 3.0 4.0}; do
  for lib in libpbp.so ${OLDLIBS:-}; do
    echo "old:$lib $e $(PBP_WS=0 PBP_LIB=$L/$lib timeout 120 python tools/prof_decode.py --n 1024 --frames 100000 --reps 3 --ebn0 $e | tail -1)"
  done
  for lib in libpbp.so ${LIBS:-}; do
    echo "$lib $e $(PBP_LIB=$L/$lib timeout 120 python tools/prof_decode.py --n 1024 --frames 100000 --reps 3 --ebn0 $e | tail -1)"
  done
done
