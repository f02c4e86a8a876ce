"""Device timeline of e2e steps (pinned-host Q/K/V, output copied back):
copies and kernels with start/end (us), compressed.  Diagnostic only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402

cfg = bench.CONFIGS[bench.DEFAULT_CONFIG]
eng, rows = bench.build_engine(cfg, 0, torch, host_inputs=True, out_len=64)
for _ in range(6):
    eng.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        eng.step()
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
last = None
for e in evs:
    n = e.name
    kind = ("H2D" if "HtoD" in n else "D2H" if "DtoH" in n else n.split("(")[0].replace("fk::", ""))
    sz = ""
    if kind in ("H2D", "D2H"):
        print(f"{kind:22s} {e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f}  dur {e.time_range.end - e.time_range.start:7.1f}")
    elif kind in ("fk_prefix_tc_kernel", "fk_append_kernel"):
        print(f"{kind:22s} {e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f}")
