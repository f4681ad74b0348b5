"""C-ABI boundary checks that need no GPU (-m "not gpu"): the library loads, exports every
symbol include/tokensim.h declares, struct layouts match the header, create() validates
its inputs with path-qualified messages, and run() fails loudly without a device."""
import ctypes as C
import os
import re
from dataclasses import replace

import pytest

import sweep_inputs as si

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def T():
    from paper_2503_08415_b200 import build
    build.build()
    from paper_2503_08415_b200 import _lib
    _lib.lib()
    return _lib


def header_functions():
    src = open(os.path.join(ROOT, "include", "tokensim.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tokensim_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(T):
    L = T.lib()
    declared = header_functions()
    assert len(declared) >= 17
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(T.EXPORTS)
    assert L.tokensim_version().decode().startswith("tokensim-b200")


def test_struct_sizes_match_header(T):
    # sizes the header documents
    assert T.RECORD_DTYPE.itemsize == 32 and T.SAMPLE_DTYPE.itemsize == 32
    assert T.ITER_DTYPE.itemsize == 80 and T.SUMMARY_DTYPE.itemsize == 384
    assert T.SUMMARY_DTYPE.fields["stat"][1] == 144 and T.SUMMARY_DTYPE.fields["throughput_rps"][1] == 344
    assert T.SUMMARY_DTYPE.fields["total_blocks"][1] == 128 and T.SUMMARY_DTYPE.fields["sched_digest"][1] == 104
    # the library itself checks struct_size: a wrong size is rejected
    from paper_2503_08415_b200.api import marshal
    cm, hws, pols, cw, co, keep = marshal(si.c1())
    cm.struct_size += 4
    h = C.c_void_p()
    st = T.lib().tokensim_sweep_create(C.byref(cm), hws, 1, pols, 1, C.byref(cw), C.byref(co), C.byref(h))
    assert st == T.E_INVALID and not h.value
    assert b"struct_size" in T.lib().tokensim_last_error(None)


def _create(cfg):
    from paper_2503_08415_b200 import Sweep
    return Sweep(cfg)


def test_create_and_grid(T):
    sw = _create(si.c3())
    assert sw.num_points == 4608
    assert sw.workspace_size() > 4608 * 10000 * 32
    sw2 = _create(si.c2())
    assert sw2.num_points == 128
    assert si.c2().point_coords(37) == (0, 0, 37 // 8, 37 % 8)


@pytest.mark.parametrize("mutate,needle", [
    (lambda c: replace(c, hws=[replace(c.hws[0], mem_capacity=10 ** 10)]), b"hw[0].mem_capacity"),
    (lambda c: replace(c, hws=[replace(c.hws[0], eff_bw=1.5)]), b"hw[0].eff_flops/eff_bw"),
    (lambda c: replace(c, policies=[si.Policy(max_num_seqs=0)]), b"policies[0].max_num_seqs"),
    (lambda c: replace(c, policies=[si.Policy(kind=si.CONT_RATIO, max_mem_ratio=0.0)]), b"max_mem_ratio"),
    (lambda c: replace(c, policies=[si.Policy(watermark_blocks=10 ** 6)]), b"watermark_blocks"),
    (lambda c: replace(c, policies=[si.Policy(max_batched_tokens=100)]), b"max_batched_tokens"),
    (lambda c: replace(c, workload=replace(c.workload, rates=[0.0])), b"workload.rates[0]"),
    (lambda c: replace(c, workload=replace(c.workload, num_requests=0)), b"num_requests"),
    (lambda c: replace(c, workload=si.Workload(2, [1.0], [0], len_dist=si.TRACE, trace_arrival_ns=[5, 1],
                                               trace_prompt=[1, 1], trace_output=[1, 1])), b"trace_arrival_ns[1]"),
    (lambda c: replace(c, workload=si.Workload(1, [1.0], [0], len_dist=si.FIXED, prompt_a=2000, output_a=100)),
     b"prompt_a/output_a"),
    # NEXT-3b: chunked prefill needs a budget >= max_num_seqs
    (lambda c: replace(c, policies=[si.Policy(iteration_mode=si.CHUNKED, max_batched_tokens=8, max_num_seqs=16)]),
     b"CHUNKED needs max_batched_tokens"),
    # NEXT-1: at most 8 workers per node; a known dispatch policy
    (lambda c: replace(c, options=si.Options(topology=si.PD_PAIR, pd_prefill=4, pd_decode=5)), b"at most 8"),
    # a.9 / NEXT-1: P/D workers are prefill-only / decode-only
    (lambda c: replace(c, policies=[si.Policy(iteration_mode=si.PREFILL_FIRST)],
                       options=si.Options(topology=si.PD_PAIR)), b"iteration_mode"),
    # NEXT-4: a preload link needs a buffer
    (lambda c: replace(c, options=si.Options(link_mode=si.PRELOAD, preload_buffer_bytes=0)), b"preload_buffer_bytes"),
    # NEXT-2: the memory cache needs multi-round conversations; those need generated lengths
    (lambda c: replace(c, options=si.Options(memory_cache=True)), b"memory_cache"),
    (lambda c: replace(c, workload=si.Workload(2, [1.0], [0], len_dist=si.TRACE, trace_arrival_ns=[0, 1],
                                               trace_prompt=[1, 1], trace_output=[1, 1], multi_round=True)),
     b"multi_round"),
])
def test_create_validation_messages(T, mutate, needle):
    from paper_2503_08415_b200 import TokensimError
    with pytest.raises(TokensimError) as ei:
        _create(mutate(si.c1()))
    assert ei.value.status == T.E_INVALID
    assert needle.decode() in str(ei.value)


def test_run_without_device_fails_loudly(T):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2503_08415_b200.api import marshal
    cm, hws, pols, cw, co, keep = marshal(si.c1())
    L = T.lib()
    h = C.c_void_p()
    assert L.tokensim_sweep_create(C.byref(cm), hws, 1, pols, 1, C.byref(cw), C.byref(co), C.byref(h)) == 0
    st = L.tokensim_sweep_run(h, 0, 0, 1, 1, None, 0, None)
    assert st == T.E_CUDA and b"no CUDA device" in L.tokensim_last_error(h)
    # getters before a successful run are state errors
    n = C.c_uint64()
    assert L.tokensim_get_summaries(h, None, 0, C.byref(n)) == T.E_STATE
    L.tokensim_sweep_destroy(h)


def test_product_does_not_import_oracle():
    """The CUDA path and the oracle share no code: no module of the product package
    mentions the oracle, and the oracle never imports the product."""
    pkg = os.path.join(ROOT, "paper_2503_08415_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
                assert "oracle.h" not in src and "liboracle" not in src, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".cpp", ".h")):
            src = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(from|import)\s+paper_2503_08415_b200", src, re.M), f
            assert not re.search(r'#include\s*[<"].*tokensim', src), f
            assert "libtokensim" not in src, f


def test_resume_checkpoint_refuses_another_sweep(T, tmp_path):
    """sweep_resumable validates its checkpoint before any device work: a checkpoint written
    for another config (or another chunking) is refused; the fingerprint is stable."""
    import numpy as np
    import paper_2503_08415_b200 as P
    a, b = si.c2(), replace(si.c2(), policies=[replace(si.c2().policies[0], max_num_seqs=128)])
    assert P.config_fingerprint(a) == P.config_fingerprint(si.c2())
    assert P.config_fingerprint(a) != P.config_fingerprint(b)
    path = str(tmp_path / "ck.npz")
    np.savez(path, fingerprint=np.array(P.config_fingerprint(b)), chunk_points=np.array(16),
             summaries=np.zeros(a.num_points * P.SUMMARY_DTYPE.itemsize, np.uint8), done=np.zeros(8, np.bool_))
    with pytest.raises(ValueError, match="another sweep"):
        P.sweep_resumable(a, path, chunk_points=16)
    np.savez(path, fingerprint=np.array(P.config_fingerprint(a)), chunk_points=np.array(32),
             summaries=np.zeros(a.num_points * P.SUMMARY_DTYPE.itemsize, np.uint8), done=np.zeros(4, np.bool_))
    with pytest.raises(ValueError, match="another sweep"):
        P.sweep_resumable(a, path, chunk_points=16)
