"""pytest plugin (diagnostic): after each test, the number of live _Pool
objects that hold a device handle, and what keeps the oldest live GpuEngine
alive (frames by code name, and who holds those frames)."""
import gc
import types


def pytest_runtest_teardown(item, nextitem):
    from paper_2405_19888_b200 import engine as E
    gc.collect()
    pools = [o for o in gc.get_objects() if isinstance(o, E._Pool) and o.handle]
    n_eng = sum(1 for o in gc.get_objects() if type(o).__name__ == "GpuEngine")
    line = f"[pool-probe] {item.nodeid} live_pools={len(pools)} engines={n_eng}"
    if len(pools) > 3:
        eng = next(o for o in gc.get_objects() if type(o).__name__ == "GpuEngine")
        frames = [r for r in gc.get_referrers(eng) if isinstance(r, types.FrameType)]
        line += " frames=" + ",".join(f.f_code.co_name for f in frames[:6])
        if frames:
            holders = [type(h).__name__ for h in gc.get_referrers(frames[0]) if h is not frames]
            line += " frame0_held_by=" + ",".join(holders[:6])
            tbs = [h for h in gc.get_referrers(frames[0]) if isinstance(h, types.TracebackType)]
            if tbs:
                owners = [type(o).__name__ for o in gc.get_referrers(tbs[0])]
                line += " tb_held_by=" + ",".join(owners[:6])
                excs = [o for o in gc.get_referrers(tbs[0]) if isinstance(o, BaseException)]
                if excs:
                    line += " exc=" + repr(excs[0])[:200]
        del eng, frames
    print(line, flush=True)
