"""GPU: a process may hold at most 64 device pools (two __constant__ plan
slots each, fk_internal.h kPlanSlots).  Engines dropped without close()
inside reference cycles keep their pool until the cycle collector runs;
creating a pool when all slots are taken collects and retries
(engine.py _Pool), so a long-lived process that creates and drops engines
does not run out."""

import gc

import pytest

import paper_2405_19888_b200 as P

from gpu_check import check_history

pytestmark = pytest.mark.gpu


def _engine(dev):
    return P.GpuEngine("e", P.CostModel(), kv_tokens=4096, device=dev, geometry=P.ModelGeometry(1, 2, 128),
                       model=P.SyntheticDecodeModel(7, 1.0), keep_history=True, capture_f32=True)


def test_dropped_engines_in_cycles_release_their_pools(cuda_device):
    gc.collect()
    gc.disable()  # only the retry in _Pool may collect
    try:
        for i in range(80):  # > 64 live pools if nothing were collected
            eng = _engine(cuda_device)
            eng._self_ref = eng  # a reference cycle: freed by the cycle collector only
            del eng
        eng = _engine(cuda_device)
        eng.fill([1] * 40, "c", None)
        eng.generate("r", "c", [1] * 2, "")
        for _ in range(2):
            eng.step()
        check_history(eng)
        eng.close()
    finally:
        gc.enable()
        gc.collect()
