"""Per-k-block clocks of CTA 0 in one GEMM launch (experiment build with
-DDASHCU_GEMM_TRACE, loaded through DASHCU_LIB_PATH): producer issue, MMA wait start,
MMA data ready, relative to the first producer issue."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17218_b200 as D  # noqa: E402
from gemm_bench import SHAPES  # noqa: E402

L = D.lib()
L.dashcu_selftest_gemm_timed.argtypes = [C.c_void_p] + [C.c_int] * 7 + [C.POINTER(C.c_double)]
ctx = D.Context(0)
for n in sys.argv[1:]:
    M, N, K, ak, bk, epi = SHAPES[n]
    ms = C.c_double(0)
    assert L.dashcu_selftest_gemm_timed(ctx.h, M, N, K, ak, bk, epi, 3, C.byref(ms)) == 0
    tr = np.zeros((3, 512), dtype=np.int64)
    assert L.dashcu_debug_gemm_trace(tr.ctypes.data_as(C.c_void_p)) == 0
    nkb = ((K + 63) // 64 + 3) // 4 if M <= 64 else (K + 63) // 64  # ring stages (4 k-blocks at M <= 64)
    nkb = min(nkb, 290)
    t = tr[:, :nkb] - tr[0, 0]
    print(n, f"{ms.value * 1e3:.2f} us/launch; k-block: producer issue / mma wait / data ready (cycles)")
    for k in list(range(0, min(nkb, 12))) + list(range(max(12, nkb - 3), nkb)):
        print(f"  {k:3d} {t[0, k]:7d} {t[1, k]:7d} {t[2, k]:7d}")
    marks = tr[2, 500:506] - tr[2, 500]
    print("  marks (cycles from kernel entry): setup done %d, pdl_wait done %d, first accumulator %d, "
          "epilogue done %d, stores drained %d; first producer issue %d"
          % (marks[1], marks[2], marks[3], marks[4], marks[5], tr[0, 0] - tr[2, 500]))
    ep = tr[2, 300:480].reshape(-1, 2) - tr[2, 500]
    ep = ep[(ep[:, 0] > 0) & (ep[:, 0] < 1e9)]
    if len(ep):
        print("  epilogue per tile (start, end, length):", [(int(a), int(b), int(b - a)) for a, b in ep[:12]])
    kbt = t[1, :nkb]
    print("  mma wait times every 14 k-blocks:", [int(x) for x in kbt[::14][:12]])
