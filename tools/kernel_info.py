"""Fast-kernel resources per code length (pbp_kernel_info): shared bytes and resident warps per SM.
   python tools/kernel_info.py"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1505_04979_b200 as P

for n in (256, 512, 1024, 2048, 4096, 8192, 16384):
    for k in (0, 1, 2):
        a, b = C.c_int32(), C.c_int32()
        P.lib.pbp_kernel_info(n, k, C.byref(a), C.byref(b))
        print(f"n={n:6d} decoder={k}: {a.value:7d} B shared, {b.value:3d} warps/SM")
