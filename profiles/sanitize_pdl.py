"""tiny config on the mma / tc prefix path with FK_OPT_PDL = argv[2] (diagnostic)."""
import os, sys
ROOT = "/root/repo"
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2405_19888_b200 as P
from paper_2405_19888_b200 import _lib
from paper_2405_19888_b200.workloads import fork_group
from gpu_check import check_history

path, pdl = sys.argv[1], int(sys.argv[2])
eng = P.GpuEngine("e0", P.CostModel(), kv_tokens=1 << 20, device=0, geometry=P.ModelGeometry(1, 32, 128),
                  model=P.SyntheticDecodeModel(0x5EED), capture_f32=True, keep_history=True)
eng.set_option(_lib.FK_OPT_TC_MIN_FANOUT, 2 if path == "tc" else 0)
eng.set_option(_lib.FK_OPT_PDL, pdl)
fork_group(eng, 1024, [64] * 8, out_len=2)
eng.step()
eng.stream.synchronize()
try:
    print(path, "pdl", pdl, "ok", check_history(eng), flush=True)
except AssertionError as e:
    print(path, "pdl", pdl, "FAIL", e, flush=True)
