"""The drop-in boundary: C ABI exports, C++ API under slabsim:: names, Python
mirror error behaviour.  CPU only (no kernel launches)."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2509_06261_b200 as ks
from paper_2509_06261_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "kvslab.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ks_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) > 40
    for s in syms:
        assert hasattr(L.lib, s), f"libkvslab.so does not export {s}"
    assert set(L.EXPORTED) >= set(syms), set(syms) - set(L.EXPORTED)
    assert L.lib.ks_abi_version() == 1


def test_status_mapping_and_messages():
    with pytest.raises(ks.InvalidConfigError):
        ks.SlabPool(ks.SlabPoolConfig(100, 0, [1]))
    p = ks.SlabPool(ks.SlabPoolConfig(4 * 65536, 65536, [32768]))
    with pytest.raises(ks.InvalidKeyError):
        p.alloc_block(1234)
    with pytest.raises(ks.InvalidFreeError):
        p.free_block(ks.BlockHandle(99, 0, 0, 32768))
    for _ in range(8):
        p.alloc_block(32768)
    assert p.try_alloc_block(32768) is None
    with pytest.raises(ks.PoolExhaustedError) as e:
        p.alloc_block(32768)
    assert "exhausted" in str(e.value)
    with pytest.raises(ks.InvalidProfileError):
        ks.token_size(9, 128, 16, tp_degree=2)


def test_host_only_pool_rejects_device_calls():
    p = ks.SlabPool(ks.SlabPoolConfig(4 * 65536, 65536, [65536]))
    base, n = C.c_void_p(), C.c_uint64()
    assert L.lib.ks_device_base(p.handle, C.byref(base), C.byref(n)) == 0 and not base.value
    assert L.lib.ks_slab_table_sync(p.handle, None) == L.KS_INVALID_ARGUMENT


def test_batched_alloc_free_and_clone():
    p = ks.SlabPool(ks.SlabPoolConfig(8 * 65536, 65536, [16384, 65536]))
    hs = p.alloc_blocks(16384, 10)
    assert [h.global_block_id for h in hs] == list(range(10))
    c = p.clone_host()
    assert c == p
    p.free_blocks(hs[:5])
    assert not (c == p)
    assert p.allocated_block_count(16384) == 5 and c.allocated_block_count() == 10


def test_cpp_dropin_compiles_and_passes(tmp_path):
    """Reference-style C++ (slabsim:: names) against libkvslab.so."""
    exe = tmp_path / "dropin"
    lib_dir = os.path.join(ROOT, "paper_2509_06261_b200")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), "-L", lib_dir,
                    "-lkvslab", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all checks passed" in out.stdout


def test_workspace_size_queries_need_no_gpu():
    """The K4 workspace size query is pure host arithmetic: split-KV partials
    when the chunk's query tiles alone would leave SMs idle, plus batch x
    bt_stride fp16 blocks (+ K scale/zero arrays) for the quantised formats."""
    from paper_2509_06261_b200.kv import KvDtype, KvFormat
    n = C.c_size_t()
    for dt in KvDtype:
        f = KvFormat(dt, 8, 32).to_c()
        # long chunks fill the GPU: no split-KV partials, only the expand scratch
        assert L.lib.ks_paged_prefill_workspace_size(C.byref(f), 4, 100, 4096, C.byref(n)) == 0
        block = 0 if dt == KvDtype.FP16 else 2 * 8 * 16 * 128 * 2 + 8 * 128
        assert n.value == 4 * 100 * block
        # one 64-token chunk: 8 CTAs -> 8 KV splits of fp32 partials (rows x 132 floats)
        assert L.lib.ks_paged_prefill_workspace_size(C.byref(f), 1, 100, 64, C.byref(n)) == 0
        assert n.value == 64 * 32 * 8 * 132 * 4 + 100 * block
    assert L.lib.ks_paged_prefill_workspace_size(None, 1, 1, 1, C.byref(n)) != 0
