"""Per-phase timeline of CTA 0 of the tcgen05 prefix kernel (debug build
with -DFK_TIMELINE, loaded via FK_LIB_PATH).  Not product code."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_19888_b200 as P  # noqa: E402
from paper_2405_19888_b200 import _lib  # noqa: E402
from paper_2405_19888_b200.workloads import fork_group  # noqa: E402

eng = P.GpuEngine("e0", P.CostModel(), kv_tokens=1 << 22, device=0, geometry=P.ModelGeometry(2, 40, 128))
eng.set_option(_lib.FK_OPT_TC_MIN_FANOUT, 2)
for kv in filter(None, os.environ.get("FK_TL_OPT", "").split(",")):  # e.g. FK_TL_OPT=TC_MIN_CHUNK=4
    k, v = kv.split("=")
    eng.set_option(getattr(_lib, "FK_OPT_" + k), int(v))
fork_group(eng, 6000, [256] * int(os.environ.get("FK_TL_FORKS", "64")), out_len=8)
for _ in range(3):
    eng.step()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 256)()
fn = _lib.lib.fk_debug_timeline
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
print("rc", fn(buf, 256))
t0 = buf[160]
names = {0: "kv_full", 16: "S_issued", 32: "p_full+o_free", 48: "PV_issued", 64: "s_full(sm)",
         80: "P_written", 96: "o_full(sm)", 112: "acc_done", 128: "kv_empty(prod)",
         176: "sm:S loaded", 192: "sm:max xchg", 208: "sm:P stored", 224: "sm:wait_st"}
print("epilogue of the first 4 pieces (read queue, O loaded, stores issued, pair barrier):")
for k in range(4):
    print("  piece", k, " ".join(f"{(buf[240 + 4 * k + j] - t0) / 1e3:7.2f}" if buf[240 + 4 * k + j] > t0 else "   -   " for j in (3, 0, 1, 2)))
for base, nm in names.items():
    print(f"{nm:16s}", " ".join(f"{(buf[base + t] - t0) / 1e3:7.2f}" if buf[base + t] > t0 else "   -   " for t in range(14)))
