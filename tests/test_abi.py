"""CPU-only checks of the C ABI: the library builds/loads, exports every symbol include/*.h
declares, and rejects bad arguments on the host before touching a device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("sfa.h", "sfa_gen.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        names |= set(re.findall(r"^SFA_API[^(]*?\b(sfa_\w+)\s*\(", src, flags=re.M))
    return names


@pytest.fixture(scope="module")
def sfa():
    from paper_2603_22300_b200 import build, sfa
    build.build()
    return sfa


def test_exports_every_declared_symbol(sfa):
    decl = declared_symbols()
    assert len(decl) >= 12
    L = sfa.lib()
    for name in decl:
        assert hasattr(L, name), name
    assert set(sfa.EXPORTS) == decl


def test_status_strings(sfa):
    s = sfa.lib().sfa_status_string
    assert [s(i).decode() for i in range(6)] == ["ok", "invalid-argument", "invalid-input", "unsupported",
                                                 "resource-limit", "cuda-error"]


def test_host_validation_before_launch(sfa):
    L = sfa.lib()
    P = ctypes.c_void_p
    dummy = P(16)
    # k out of range -> invalid-argument; d not compiled -> unsupported
    assert L.sfa_topk_codes(dummy, 1, 10, 128, 128, 0, dummy, dummy, None, None) == 1
    assert L.sfa_topk_codes(dummy, 1, 10, 128, 128, 129, dummy, dummy, None, None) == 1
    assert L.sfa_topk_codes(dummy, 1, 10, 96, 96, 8, dummy, dummy, None, None) == 3
    assert L.sfa_topk_codes(dummy, 7, 10, 128, 128, 8, dummy, dummy, None, None) == 1
    assert L.sfa_topk_codes(None, 1, 10, 128, 128, 8, dummy, dummy, None, None) == 1
    assert L.sfa_topk_codes(dummy, 1, 0, 128, 128, 8, None, None, None, None) == 0  # empty is ok
    # the fused Q + K launch validates both tensors before any launch
    qk = L.sfa_topk_codes_qk
    assert qk(dummy, 10, 128, dummy, dummy, dummy, 10, 128, dummy, dummy, 1, 128, 0, None, None) == 1   # k = 0
    assert qk(dummy, 10, 128, dummy, dummy, dummy, 10, 64, dummy, dummy, 1, 128, 8, None, None) == 1   # K ld < d
    assert qk(dummy, 10, 128, dummy, dummy, None, 10, 128, dummy, dummy, 1, 128, 8, None, None) == 1   # K null
    assert qk(dummy, 10, 96, dummy, dummy, dummy, 10, 96, dummy, dummy, 1, 96, 8, None, None) == 3     # d = 96
    assert qk(dummy, 0, 128, None, None, dummy, 0, 128, None, None, 1, 128, 8, None, None) == 0      # empty


def desc(sfa, **kw):
    base = dict(B=1, H=4, H_kv=2, d=128, k=16, d_v=128, n_q=300, n_kv=300)
    base.update(kw)
    return sfa.make_desc(**base)


def test_desc_validation(sfa):
    L = sfa.lib()
    ok = desc(sfa, kernel=sfa.KERNEL_SIMT)
    assert L.sfa_attn_workspace_bytes(ctypes.byref(ok)) > 0
    # the default sm_100a kernel (SM100_OT, no buckets): the 256-aligned max|V| per (b, kv head) + the
    # fp16 copy of V (reading A12), then 256-aligned, the decompressed bf16 K~ rows its TMA reads, then
    # 256 bytes for the persistent tile scheduler's work counter
    v16 = 256 + 1 * 2 * 300 * 128 * 2
    kd = 1 * 2 * 300 * 128 * 2
    assert L.sfa_attn_workspace_bytes(ctypes.byref(desc(sfa))) == \
        (v16 + 255) // 256 * 256 + (kd + 255) // 256 * 256 + 256
    # SM100 (d_v = 64 default) decompresses the key codes on chip: V prep only
    assert L.sfa_attn_workspace_bytes(ctypes.byref(desc(sfa, kernel=sfa.KERNEL_SM100))) == v16
    bad = [dict(H=3, H_kv=2), dict(k=0), dict(k=129), dict(n_q=0), dict(n_kv=0), dict(scale=-1.0),
           dict(scale=float("inf")), dict(q_pos0=-1)]
    for b in bad:
        d = desc(sfa, **b)
        assert L.sfa_attn_workspace_bytes(ctypes.byref(d)) == 0, b
        assert L.sfa_attn_fwd(ctypes.byref(d), *([ctypes.c_void_p(16)] * 8), 1 << 30, None) == 1, b
    for b in (dict(d=96, k=8), dict(d_v=96), dict(dtype=sfa.SFA_F32, kernel=sfa.KERNEL_SM100)):
        d = desc(sfa, **b)
        assert L.sfa_attn_fwd(ctypes.byref(d), *([ctypes.c_void_p(16)] * 8), 1 << 30, None) == 3, b
    # workspace too small -> resource-limit
    assert L.sfa_attn_fwd(ctypes.byref(ok), *([ctypes.c_void_p(16)] * 8), 16, None) == 4
    # misaligned pointers -> invalid-argument
    assert L.sfa_attn_fwd(ctypes.byref(ok), *([ctypes.c_void_p(18)] * 8), 1 << 30, None) == 1


def test_workspace_layout(sfa):
    """Key-tile bucket layout: per (b, kv head, tile) off[d+1] u16 (16-aligned) +
    (BK*k + 3d rounded to 4) entries of 4 B (bf16) or 8 B (fp32)."""
    L = sfa.lib()
    for (k, bk) in ((8, 128), (16, 128), (32, 128), (64, 64), (128, 64)):
        for dt, eb in ((sfa.SFA_BF16, 4), (sfa.SFA_F32, 8)):
            d = desc(sfa, k=k, dtype=dt, kernel=sfa.KERNEL_SIMT)
            assert L.sfa_key_tile(ctypes.byref(d)) == bk
            off = (129 * 2 + 15) // 16 * 16
            cap = (bk * k + 3 * 128 + 3) // 4 * 4
            tile = (off + cap * eb + 15) // 16 * 16
            ntiles = (300 + bk - 1) // bk
            assert L.sfa_attn_workspace_bytes(ctypes.byref(d)) == 1 * 2 * ntiles * tile


def test_bucketed_entry_points_need_simt(sfa):
    """sfa_bucket_keys / sfa_attn_fwd_bucketed feed the CUDA-core kernel only (unsupported otherwise)."""
    L = sfa.lib()
    d = desc(sfa, kernel=sfa.KERNEL_SM100)
    assert L.sfa_bucket_keys(ctypes.byref(d), *([ctypes.c_void_p(16)] * 3), 1 << 30, None) == 3
    assert L.sfa_attn_fwd_bucketed(ctypes.byref(d), *([ctypes.c_void_p(16)] * 6), 1 << 30, None) == 3


def test_n4_semantics_validation(sfa):
    """edges_only (R2) and window (sliding window) are validated on the host before any launch and
    select the OT / SIMT kernels; the R2 workspace adds the per-tile feature bitsets (edges.cu)."""
    L = sfa.lib()
    base = L.sfa_attn_workspace_bytes(ctypes.byref(desc(sfa)))
    r2 = L.sfa_attn_workspace_bytes(ctypes.byref(desc(sfa, edges_only=True)))
    ntiles = (300 + 127) // 128
    assert r2 == (base + 255) // 256 * 256 + 1 * 2 * ntiles * 128 * 16  # [B*H_kv][tiles][d][4] u32
    assert L.sfa_attn_workspace_bytes(ctypes.byref(desc(sfa, window=64))) == base  # window: no extra state
    for b in (dict(window=-1), dict(window=16, causal=False)):
        d = desc(sfa, **b)
        assert L.sfa_attn_fwd(ctypes.byref(d), *([ctypes.c_void_p(16)] * 8), 1 << 30, None) == 1, b
    # block selection (N4): argument and support checks before any launch
    bsf = L.sfa_attn_fwd_blocksel
    dv16 = ctypes.c_void_p(16)
    assert bsf(ctypes.byref(desc(sfa)), *([dv16] * 6), 0, dv16, dv16, dv16, 1 << 30, None) == 1        # max_sel 0
    assert bsf(ctypes.byref(desc(sfa)), *([dv16] * 5), None, 4, dv16, dv16, dv16, 1 << 30, None) == 1   # no list
    for b in (dict(H=6, H_kv=2), dict(edges_only=True), dict(window=64), dict(d_v=64),
              dict(dtype=sfa.SFA_F32), dict(kernel=sfa.KERNEL_SM100_PP)):
        assert bsf(ctypes.byref(desc(sfa, **b)), *([dv16] * 6), 4, dv16, dv16, dv16, 1 << 30, None) == 3, b
    assert bsf(ctypes.byref(desc(sfa)), *([dv16] * 6), 4, dv16, dv16, dv16, 16, None) == 4             # workspace
    # d_v = 64 runs when the desc names SM100_OT (AUTO picks SM100 for d_v = 64): it gets to the workspace check
    d64 = desc(sfa, d_v=64, kernel=sfa.KERNEL_SM100_OT)
    assert bsf(ctypes.byref(d64), *([dv16] * 6), 4, dv16, dv16, dv16, 16, None) == 4
    # the round-1 ablation kernels PAIR / WIDE were removed in round 2: their numbers stay reserved
    for kern in (sfa.KERNEL_SM100_PAIR, sfa.KERNEL_SM100_WIDE):
        assert L.sfa_attn_fwd(ctypes.byref(desc(sfa, kernel=kern)), *([ctypes.c_void_p(16)] * 8), 1 << 30, None) == 3
    for kern in (sfa.KERNEL_SM100, sfa.KERNEL_SM100_PAIR, sfa.KERNEL_SM100_WIDE, sfa.KERNEL_DECODE,
                 sfa.KERNEL_SM100_PP, sfa.KERNEL_SM100_OTH):
        for b in (dict(edges_only=True), dict(window=16)):
            d = desc(sfa, kernel=kern, **b)
            assert L.sfa_attn_fwd(ctypes.byref(d), *([ctypes.c_void_p(16)] * 8), 1 << 30, None) == 3, (kern, b)
    # the fused step-1-on-Q entry needs the OT kernel with R1 and no window
    for b in (dict(edges_only=True), dict(window=16), dict(d_v=64)):
        d = desc(sfa, **b)
        assert L.sfa_attn_fwd_fused_q(ctypes.byref(d), *([ctypes.c_void_p(16)] * 9), ctypes.c_void_p(16),
                                      1 << 30, None) == 3, b
    # the backward covers R1 without a window
    for b in (dict(edges_only=True), dict(window=16)):
        d = desc(sfa, **b)
        assert L.sfa_attn_bwd(ctypes.byref(d), *([ctypes.c_void_p(16)] * 12), 1 << 30, None) == 3, b
