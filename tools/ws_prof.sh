for e in ${@:-1.0 3.0}; do echo "== $e"
PBP_LIB=$PWD/paper_1505_04979_b200/_lib/libpbp_prof.so timeout 120 python tools/prof_decode.py --n 1024 --frames 100000 --reps 1 --ebn0 $e | tail -14
done
