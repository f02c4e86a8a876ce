"""Layer time by launch path (diagnostic): the engine's own step graph
(fk_attn_decode_layers) vs a torch-captured graph of per-layer fk_attn_decode
calls, each at PDL level 1 and 2, and the isolated sequence (a foreign
kernel between layers).  Interleaved rounds; prints median us per layer.

    python profiles/graph_ab.py [--config ...] [--rounds 5]
"""
import argparse
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2405_19888_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=bench.DEFAULT_CONFIG)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    eng, rows = bench.build_engine(cfg, 0, torch, out_len=64)
    for _ in range(4):
        eng.step()
    torch.cuda.synchronize()
    L, H = cfg["L"], cfg["H"]
    q = eng.model.q
    out = torch.empty_like(q)
    le = rows * H * 128 * 2
    st = eng.stream
    sp = ctypes.c_void_p(st.cuda_stream)
    h = eng._pool.handle
    foreign = torch.empty(1 << 16, dtype=torch.float32, device=q.device)

    def engine_graph():
        _lib.check(_lib.lib.fk_attn_decode_layers(h, 0, L, ctypes.c_void_p(q.data_ptr()), le,
                                                  ctypes.c_void_p(out.data_ptr()), le, None, 0, sp))

    def per_layer(with_foreign):
        def f():
            for layer in range(L):
                if with_foreign:
                    foreign.add_(1.0)
                _lib.check(_lib.lib.fk_attn_decode(h, layer, ctypes.c_void_p(q.data_ptr() + layer * le),
                                                   ctypes.c_void_p(out.data_ptr() + layer * le), None, sp))
        return f

    def capture(fn):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            fn()
            st.synchronize()
            with torch.cuda.graph(g, stream=st):
                fn()
        return g

    def time(fn):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):  # graph replays go to the current stream
            fn()
            s.record(st)
            for _ in range(args.reps):
                fn()
            e.record(st)
            e.synchronize()
        return s.elapsed_time(e) * 1e3 / (args.reps * L)

    variants = {}
    for pdl in (1, 2):
        eng.set_option(_lib.FK_OPT_PDL, pdl)
        variants[f"engine graph PDL={pdl}"] = (pdl, engine_graph)
        g = capture(per_layer(False))
        variants[f"torch graph PDL={pdl}"] = (pdl, g.replay)
        gf = capture(per_layer(True))
        variants[f"torch graph + foreign PDL={pdl}"] = (pdl, gf.replay)
    eng.set_option(_lib.FK_OPT_PDL, 1)
    gfo = capture(lambda: [foreign.add_(1.0) for _ in range(L)])
    variants["foreign only"] = (1, gfo.replay)
    res = {k: [] for k in variants}
    for _ in range(args.rounds):
        for name, (pdl, fn) in variants.items():
            eng.set_option(_lib.FK_OPT_PDL, pdl)
            res[name].append(time(fn))
    for name, v in res.items():
        print(f"{name:34s} {statistics.median(v):7.2f} us/layer  ({', '.join(f'{x:.2f}' for x in v)})", flush=True)


if __name__ == "__main__":
    main()
