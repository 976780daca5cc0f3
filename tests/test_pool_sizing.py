"""a4 -- the reference's per-GPU-group pool sizing (simulator.cpp:264-290,
precision.cpp:119-127) restated in paper_2509_06261_b200/placement.py,
against golden vectors the compiled reference produced for every shipped
scenario (tests/golden/pool_sizing.json, oracle/make_golden.py pool_sizing)."""
import json
import os

import pytest

import paper_2509_06261_b200 as ks
from paper_2509_06261_b200.placement import (ResidentModel, lcm_slab_bytes, residual_pool_bytes)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pool_sizing.json")))


@pytest.mark.parametrize("sc", GOLD["scenarios"], ids=[s["scenario"] for s in GOLD["scenarios"]])
def test_pool_and_slab_sizes_match_the_reference(sc):
    for g in sc["groups"]:
        ms = [ResidentModel(m["model"], m["key"], m["weight_bytes"], m["operating_batch"], m["tp_degree"],
                            m["avg_activation_bytes"], m["avg_kv_bytes"]) for m in g["models"]]
        pool = residual_pool_bytes(ms, g["total_memory"]) if sc["residual"] else sc["explicit_pool"]
        assert pool == g["pool_bytes"], (sc["scenario"], g["group"])
        keys = sorted({m.key for m in ms})
        slab = lcm_slab_bytes(keys, sc["slab_multiplier"]) if sc["slab_auto_lcm"] else sc["slab_explicit"]
        assert slab == g["slab_size_bytes"], (sc["scenario"], g["group"])
        # and the allocator accepts that geometry exactly like the reference's
        pool_obj = ks.SlabPool(ks.SlabPoolConfig(pool, slab, keys, sc["slab_auto_lcm"]))
        assert pool_obj.slab_count() == pool // slab


def test_footprints_beyond_memory_are_rejected():
    m = ResidentModel("m", 65536, 10 << 30, 8, 1, 1 << 20, 1 << 20)
    with pytest.raises(ValueError):
        residual_pool_bytes([m], 4 << 30)


@pytest.mark.gpu
def test_device_pool_from_the_gpus_memory():
    """The same policy on a B200: group memory = the device's, the pool bounded
    by its free memory; the pool is created and every key allocates."""
    import torch
    from paper_2509_06261_b200.kv import KvDtype, KvFormat
    from paper_2509_06261_b200.placement import device_pool_config
    fmts = [KvFormat(dt, 8, 32, num_layers=32) for dt in (KvDtype.FP16, KvDtype.INT4)]
    ms = [ResidentModel(f"m{i}", f.key, 16 << 30 if i == 0 else 5 << 30, 32, 1, 64 << 20, 256 << 20)
          for i, f in enumerate(fmts)]
    cfg = device_pool_config(ms, device=0)
    free, total = torch.cuda.mem_get_info(0)
    assert cfg.capacity_bytes <= free and cfg.capacity_bytes % cfg.slab_size_bytes == 0
    assert cfg.capacity_bytes <= residual_pool_bytes(ms, total)
    pool = ks.SlabPool(cfg, device=0)
    for f in fmts:
        assert pool.try_alloc_block(f.key) is not None
    del pool
