"""Bisect the co-run parity failure (diagnostic only)."""
import os, sys
ROOT = "/root/repo"
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2405_19888_b200 as P
from paper_2405_19888_b200 import _lib
from paper_2405_19888_b200.workloads import fork_group
from gpu_check import check_history


def run(corun, target, order=0, H=32, pdl=1, plen=1024, n=8, slen=64):
    eng = P.GpuEngine("e0", P.CostModel(), kv_tokens=1 << 20, device=0, geometry=P.ModelGeometry(1, H, 128),
                      model=P.SyntheticDecodeModel(0x5EED), capture_f32=True, keep_history=True)
    eng.set_option(_lib.FK_OPT_TC_MIN_FANOUT, 2)
    eng.set_option(_lib.FK_OPT_CORUN, corun)
    eng.set_option(_lib.FK_OPT_LAUNCH_ORDER, order)
    eng.set_option(_lib.FK_OPT_PDL, pdl)
    if target:
        eng.set_option(_lib.FK_OPT_PREFIX_TARGET_CTAS, target)
    fork_group(eng, plen, [slen] * n, out_len=2)
    eng.step()
    eng.stream.synchronize()
    try:
        w = check_history(eng)
        res = "ok %s" % w
    except AssertionError as e:
        res = "FAIL %s" % (e,)
    print(f"corun={corun} target={target} order={order} H={H} pdl={pdl} ctas={eng.last_plan.num_prefix_ctas} slots={eng.last_plan.max_slots}: {res}", flush=True)
    eng.close()


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(*[int(x) for x in sys.argv[1:]])
    else:
        for args in [(0, 106, 0, 32, 1), (0, 106, 0, 32, 0), (1, 0, 0, 32, 0), (0, 106, 0, 4, 1), (0, 7, 0, 32, 1), (0, 7, 0, 32, 0)]:
            run(*args)
