"""Create and drop 80 small device engines (close() or plain del), then one
more; prints how far it got (diagnostic for the per-process pool limit under
compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import paper_2405_19888_b200 as P  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "close"
for i in range(80):
    try:
        e = P.GpuEngine("e", P.CostModel(), kv_tokens=4096, device=0, geometry=P.ModelGeometry(1, 2, 128),
                        model=P.SyntheticDecodeModel(7, 1.0))
    except Exception as ex:
        print(mode, "failed at", i, ex)
        break
    if mode == "close":
        e.close()
    del e
else:
    print(mode, "created 80")
