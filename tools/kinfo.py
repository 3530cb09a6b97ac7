"""Fast-kernel resources per code length: python tools/kinfo.py [n ...] (library from PBP_LIB)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1505_04979_b200 as P
for n in [int(x) for x in (sys.argv[1:] or ["1024", "2048", "4096", "8192", "16384"])]:
    for kind in (0, 1, 2):
        sm, w = C.c_int32(), C.c_int32()
        P.lib.pbp_kernel_info(n, kind, C.byref(sm), C.byref(w))
        print(f"n={n} kind={kind} smem={sm.value} warps/SM={w.value} cluster={P.lib.pbp_kernel_cluster(n, kind)}")
