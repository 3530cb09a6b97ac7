# A/B of library builds (LIBS, in paper_1505_04979_b200/_lib) on csfg decodes at NS (prof_decode.py)
set -u
L=$PWD/paper_1505_04979_b200/_lib
for n in ${NS:-4096 8192 16384}; do
  f=$((40000*1024/n)); [ $f -lt 4440 ] && f=4440
  for e in ${EBN0:-2.5}; do for lib in ${LIBS:-libpbp.so}; do
    echo "$lib n=$n $e $(PBP_LIB=$L/$lib timeout 300 python tools/prof_decode.py --n $n --kind ${KIND:-csfg} --ebn0 $e --frames $f --reps 3 2>&1 | tail -1)"
  done; done
done
