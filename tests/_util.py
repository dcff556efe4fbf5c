"""Test helpers: device payload <-> oracle's unpacked (codes, scales) representation."""
from __future__ import annotations

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1
GAMMA_INV = pow(GOLDEN, -1, 1 << 64)


def draws_between(s0: int, s1: int) -> int:
    """Number of next_u64 calls that took state s0 to s1 (state += gamma per draw)."""
    return ((s1 - s0) * GAMMA_INV) & M64


def unpack_codes(buf: np.ndarray, count: int, q: int) -> np.ndarray:
    """Inverse of pack_codes (compress.cpp:352-391): q-bit two's complement, LSB first."""
    nbytes = (count * q + 7) // 8
    bits = np.unpackbits(buf[:nbytes], bitorder="little")[: count * q].reshape(count, q)
    u = (bits.astype(np.int64) << np.arange(q)).sum(1)
    u = np.where(u & (1 << (q - 1)), u - (1 << q), u)
    return u.astype(np.int8)


def decode_payload(layout, payload, rank: int, q: int):
    """Device payload -> (codes, scales) in the oracle's unpacked layout."""
    host = payload.detach().cpu().numpy() if hasattr(payload, "detach") else np.asarray(payload)
    host = host.astype(np.uint8, copy=False)
    seg = layout.segments(rank, q)
    codes, scales = [], []
    for i, s in enumerate(layout.shapes):
        if len(s) == 2:
            a, b = s
            r = min(rank, a, b)
            codes.append(unpack_codes(host[seg[i, 0]:], a * r, q))
            codes.append(unpack_codes(host[seg[i, 1]:], b * r, q))
            scales.append(host[seg[i, 2]:seg[i, 2] + 4 * r].view(np.float32))
            scales.append(host[seg[i, 3]:seg[i, 3] + 4 * r].view(np.float32))
        else:
            codes.append(unpack_codes(host[seg[i, 0]:], s[0], q))
            scales.append(host[seg[i, 2]:seg[i, 2] + 4].view(np.float32))
    return np.concatenate(codes), np.concatenate(scales)


def split_q(shapes, rank, qflat):
    """Oracle Q factor concatenation (b x r row-major per 2-D tensor) -> list."""
    out, o = [], 0
    for s in shapes:
        if len(s) != 2:
            continue
        b, r = s[1], min(rank, *s)
        out.append(qflat[o:o + b * r].reshape(b, r))
        o += b * r
    return out


def split_dense(shapes, flat):
    out, o = [], 0
    for s in shapes:
        n = int(np.prod(s))
        out.append(flat[o:o + n].reshape(s))
        o += n
    return out


def rel_fro(a, b) -> float:
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a - b))
