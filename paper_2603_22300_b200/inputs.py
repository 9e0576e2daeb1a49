"""Seeded synthetic inputs (host side) -- shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no top-k, no scores, no softmax): it only
draws the dense Q, K, V the method consumes.  It is a counter-based generator, so any
element of any tensor can be regenerated independently (the oracle can check sampled rows
of a 32K-1M token run without copying the tensors back), and it is bit-identical to the
device generator ``sfa_gen_fill`` in csrc/gen.cu (checked by tests/test_gpu_gen.py).

Recipe:
    h  = splitmix64(seed * 0x100000001B3  XOR  tensor_id << 56  XOR  flat_index)
    z  = (sum of the four 16-bit lanes of h) - 131070          # Irwin-Hall(4), integer
    x  = z * 2**-15                                             # exact in fp32, std ~1.155
    bf16(x) = round-to-nearest-even of the fp32 bit pattern     # A21
Variants: "iid" (above); "lattice" (x = (h mod 9) - 4, integer ties everywhere, for the
tie-break pins); "skewed": x * 2**e_u with an integer exponent per (head, feature),
e_u = (h' mod (2*S+1)) - S drawn from tensor id 8+tensor_id, so the products stay exact in
fp32 and the top-k index usage is unbalanced (normalised index entropy < 1).
"""
from __future__ import annotations

import numpy as np

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)
TID_Q, TID_K, TID_V, TID_DO = 1, 2, 3, 4  # TID_DO: upstream gradient dO of the backward


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x += np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def _hash(seed: int, tensor_id: int, flat: np.ndarray) -> np.ndarray:
    base = np.uint64((seed * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF) ^ np.uint64((tensor_id & 0xFF) << 56)
    return splitmix64(base ^ flat.astype(np.uint64))


def _irwin_hall_f32(h: np.ndarray) -> np.ndarray:
    m = np.uint64(0xFFFF)
    z = ((h & m) + ((h >> np.uint64(16)) & m) + ((h >> np.uint64(32)) & m) + (h >> np.uint64(48))).astype(np.int64)
    z -= 131070
    return (z.astype(np.float32) * np.float32(2.0 ** -15)).astype(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (uint16).  Inputs here are finite."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def gen_f32(seed: int, tensor_id: int, shape, *, variant: str = "iid", flat: np.ndarray | None = None,
            skew_span: int = 3) -> np.ndarray:
    """fp32 values of tensor ``tensor_id`` (shape [..., H, n, d] for skew) at the given flat indices.

    ``flat``: optional int64 flat indices into ``shape`` (default: the whole tensor).
    """
    shape = tuple(int(s) for s in shape)
    if flat is None:
        flat = np.arange(int(np.prod(shape)), dtype=np.int64)
        out_shape = shape
    else:
        flat = np.asarray(flat, dtype=np.int64)
        out_shape = flat.shape
    h = _hash(seed, tensor_id, flat.reshape(-1))
    if variant == "iid":
        x = _irwin_hall_f32(h)
    elif variant == "lattice":
        x = ((h % np.uint64(9)).astype(np.int64) - 4).astype(np.float32)
    elif variant == "skewed":
        x = _irwin_hall_f32(h)
        d = shape[-1]
        n = shape[-2]
        feat = flat.reshape(-1) % d
        head = flat.reshape(-1) // (d * n)  # flat (b, h) head id
        g = _hash(seed, 8 + tensor_id, head * d + feat)
        e = (g % np.uint64(2 * skew_span + 1)).astype(np.int64) - skew_span
        x = (x * np.exp2(e).astype(np.float32)).astype(np.float32)  # exact: power-of-two gain
    else:
        raise ValueError(variant)
    return x.reshape(out_shape)


def gen(seed: int, tensor_id: int, shape, dtype: str, **kw) -> np.ndarray:
    """Tensor in the path's storage dtype: float32 array, or uint16 bf16 bit patterns."""
    x = gen_f32(seed, tensor_id, shape, **kw)
    if dtype == "f32":
        return x
    if dtype == "bf16":
        return f32_to_bf16_bits(x)
    raise ValueError(dtype)


def qkv(seed: int, B: int, H: int, H_kv: int, n: int, d: int, d_v: int, dtype: str, variant: str = "iid",
        n_kv: int | None = None):
    """Dense Q [B,H,n,d], K [B,H_kv,n_kv,d], V [B,H_kv,n_kv,d_v] for one config."""
    n_kv = n if n_kv is None else n_kv
    q = gen(seed, TID_Q, (B, H, n, d), dtype, variant=variant)
    k = gen(seed, TID_K, (B, H_kv, n_kv, d), dtype, variant=variant)
    v = gen(seed, TID_V, (B, H_kv, n_kv, d_v), dtype, variant="iid" if variant == "skewed" else variant)
    return q, k, v
