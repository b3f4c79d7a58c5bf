"""GPU: the split fp32 master of the single-replica fused update.

The fused wgrad + SGD kernel keeps the fp32 master m as its bf16 rounding W (the weights the
GEMMs read anyway) plus lo = the low 16 bits of m, so an update moves 8 B per parameter
instead of 10.  The restatement below (numpy, bit arithmetic) is the checker:

  split: W = RNE_bf16(m), lo = m & 0xFFFF, except a tie RNE rounds up (lo == 0x8000 with an odd
         high half) is stored as lo = 0x8001 (one fp32 ulp up; W unchanged)
  join:  m = ((W - (lo > 0x8000)) << 16) | lo

The update itself is the fp32 one of trainer.cpp:56-61 (m -= scale * bf16(g), W = RNE(m)), so
the split kernel must give the same W bits as the fp32-master kernel and the same master up
to the one-ulp tie nudges.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def split_np(bits):
    bits = bits.astype(np.uint64)
    hi = bits >> 16
    lo = bits & 0xFFFF
    up = (lo > 0x8000) | ((lo == 0x8000) & ((hi & 1) == 1))
    w = (hi + up.astype(np.uint64)) & 0xFFFF
    lo = np.where((lo == 0x8000) & ((hi & 1) == 1), 0x8001, lo)
    return w.astype(np.uint16), lo.astype(np.uint16)


def join_np(w, lo):
    w = w.astype(np.uint64)
    lo = lo.astype(np.uint64)
    hi = (w - (lo > 0x8000).astype(np.uint64)) & 0xFFFF
    return ((hi << 16) | lo).astype(np.uint32)


@pytest.fixture(scope="module")
def L():
    import torch
    torch.cuda.set_device(0)
    from paper_1909_11985_b200 import _lib
    return _lib.lib()


def _s():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def test_split_join_bits_match_restatement(L):
    import torch
    rng = np.random.default_rng(5)
    bits = rng.integers(0, 2**32, size=1 << 20, dtype=np.uint64).astype(np.uint32)
    # finite values only (exponent != 0xFF), plus the edge cases by construction
    bits = bits[((bits >> 23) & 0xFF) != 0xFF]
    hi = rng.integers(0, 0x7F7F, size=4096, dtype=np.uint64).astype(np.uint32)
    edge = np.concatenate([
        (hi << 16) | 0x8000,                       # ties, both parities of hi
        (hi << 16) | 0x8000 | 0x80000000,          # negative ties
        (hi << 16) | 0x7FFF, (hi << 16) | 0x8001,  # just below / above a tie
        np.array([0, 0x80000000, 1, 0x8000, 0x18000, 0x80008000, 0x7F7FFFFF, 0xFF7FFFFF,
                  0x00010000, 0x007FFFFF], dtype=np.uint32)]).astype(np.uint32)
    bits = np.concatenate([bits, edge])
    m = torch.from_numpy(bits.view(np.float32).copy()).cuda()
    n = m.numel()
    lo = torch.empty(n, dtype=torch.int16, device="cuda")
    W = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    assert L.edl_master_split(C.c_void_p(m.data_ptr()), C.c_void_p(lo.data_ptr()),
                              C.c_void_p(W.data_ptr()), n, _s()) == 0
    back = torch.empty_like(m)
    assert L.edl_master_join(C.c_void_p(W.data_ptr()), C.c_void_p(lo.data_ptr()),
                             C.c_void_p(back.data_ptr()), n, _s()) == 0
    torch.cuda.synchronize()
    w_np, lo_np = split_np(bits)
    got_w = W.view(torch.int16).cpu().numpy().view(np.uint16)
    got_lo = lo.cpu().numpy().view(np.uint16)
    np.testing.assert_array_equal(got_w, w_np)
    np.testing.assert_array_equal(got_lo, lo_np)
    # W is torch's own RNE bf16 of m
    assert torch.equal(W, m.to(torch.bfloat16))
    got = back.cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(got, join_np(w_np, lo_np))
    tie_up = ((bits & 0xFFFF) == 0x8000) & (((bits >> 16) & 1) == 1)
    np.testing.assert_array_equal(got[~tie_up], bits[~tie_up])          # lossless ...
    np.testing.assert_array_equal(got[tie_up], bits[tie_up] | 1)        # ... but the nudged ties
    print(f"split/join: {n} values, {int(tie_up.sum())} rounded-up ties nudged by one ulp")


@pytest.mark.parametrize("M,N,K", [(1024, 768, 512), (512, 4096, 256)])
def test_split_fused_update_matches_fp32_master(L, M, N, K):
    """Modes 3 (fp32 master in, split out), 1 (split in / out) and 2 (split in, fp32 master
    out), as the job runs them around a switch, against the fp32-master kernel."""
    import torch
    torch.manual_seed(M + N)
    acts = [torch.randn(K, max(M, N)).to(torch.bfloat16).cuda() for _ in range(2)]
    dy, x = acts[0][:, :M].contiguous(), acts[1][:, :N].contiguous()
    m32 = (torch.randn(M, N, device="cuda") * 0.05).contiguous()
    W32 = m32.to(torch.bfloat16)
    ms = m32.clone()  # the split path's fp32 master (read by mode 3, written by mode 2)
    Wl = W32.clone()
    lo = torch.empty(M, N, dtype=torch.int16, device="cuda")
    joined = torch.empty_like(m32)
    P = lambda t: C.c_void_p(t.data_ptr())
    for step, mode in enumerate([3, 1, 1, 2, 3, 1, 2]):
        scale = C.c_float(2e-3)
        assert L.edl_gemm_wgrad_sgd(P(dy), M, P(x), N, P(m32), P(W32), N, M, N, K, scale,
                                    _s()) == 0
        assert L.edl_gemm_wgrad_sgd_split(P(dy), M, P(x), N, P(lo), P(Wl), P(ms), mode, N,
                                          M, N, K, scale, _s()) == 0
        if mode == 2:
            joined.copy_(ms)
        else:
            assert L.edl_master_join(P(Wl), P(lo), P(joined), M * N, _s()) == 0
        torch.cuda.synchronize()
        w_bad = (Wl.view(torch.int16) != W32.view(torch.int16))
        m_bad = joined != m32
        # a nudge is one ulp of the element at the time; later updates may shrink the element,
        # so bound the difference by the ulps of the largest magnitude
        rel = ((joined - m32).abs().max() / m32.abs().max()).item()
        print(f"step {step} mode {mode}: W mismatches {int(w_bad.sum())}, master mismatches "
              f"{int(m_bad.sum())} of {M * N}, max |diff| / max |m| {rel:.2e}")
        # the nudged ties are ~2^-16 of the values; the trajectories they start differ by
        # a few fp32 ulps and almost never cross a bf16 rounding boundary
        assert int(w_bad.sum()) <= max(2, M * N // 100000)
        assert int(m_bad.sum()) <= M * N // 1024
        assert rel <= 2.0 ** -21
    # argument checks: modes 2 / 3 need the fp32 master, unknown modes are refused
    assert L.edl_gemm_wgrad_sgd_split(P(dy), M, P(x), N, P(lo), P(Wl), None, 2, N, M, N, K,
                                      C.c_float(0.0), _s()) == 2
    assert L.edl_gemm_wgrad_sgd_split(P(dy), M, P(x), N, P(lo), P(Wl), P(ms), 4, N, M, N, K,
                                      C.c_float(0.0), _s()) == 2


def test_split_fused_update_a_resident_variant():
    """The opt-in A-resident kernel (EDL_SGD_ARES=1: the dY panel of a row block stays in
    shared memory, only X streams) runs the same checks; the switch is read once per process,
    so the checks run in a child process."""
    import os
    import subprocess
    import sys
    if os.environ.get("EDL_SGD_ARES") == "1":
        pytest.skip("already the A-resident variant")
    env = dict(os.environ, EDL_SGD_ARES="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-k",
                        "matches_fp32_master", os.path.abspath(__file__)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
