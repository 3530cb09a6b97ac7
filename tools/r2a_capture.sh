set -u
O=gpurun_out; mkdir -p $O
nvidia-smi > $O/r2a_smi.txt 2>&1
python -m pytest tests -m gpu -x -q > $O/r2a_gputest.log 2>&1; echo "gputest rc=$?"
for e in 1.0 3.0 4.0; do python tools/prof_decode.py --n 1024 --frames 100000 --reps 2 --ebn0 $e | tail -1; done > $O/r2a_points.txt 2>&1
python tools/prof_decode.py --n 1024 --frames 100000 --reps 2 --ebn0 3.0 --kind baseline | tail -1 >> $O/r2a_points.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:bp_warp_kernel -c 1 -o $O/r2a_prof_csfg python tools/prof_decode.py --n 1024 --frames 20000 --reps 1 > $O/r2a_ncu_csfg.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --import-source on --clock-control none -k regex:bp_cta_kernel -c 1 -o $O/r2a_prof_cta4096 python tools/prof_decode.py --n 4096 --frames 4000 --reps 1 --ebn0 2.5 > $O/r2a_ncu_cta4096.log 2>&1; echo "ncu2 rc=$?"
ncu --set full --import-source on --clock-control none -k regex:bp_cta_kernel -c 1 -o $O/r2a_prof_cta16384 python tools/prof_decode.py --n 16384 --frames 600 --reps 1 --ebn0 2.5 > $O/r2a_ncu_cta16384.log 2>&1; echo "ncu3 rc=$?"
