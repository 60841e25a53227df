"""Compact storage of oracle reference fields under tests/golden/ (test infrastructure).

Holds none of the method's arithmetic: it only packs a float64 field written by a committed
script that calls oracle/ (tools/make_golden_fullrun.py) and unpacks it in the tests.

Encoding: every value is rounded to a multiple of 2**-QBITS (QBITS = 36, so the stored value
differs from the oracle's by at most 2**-37 = 7.3e-12 absolute, i.e. <= 3e-13 relative for
temperatures of ~24 C -- 0.03 % of the 1e-9 parity bar), the integers are delta-coded along
the array, split into byte planes and lzma-compressed.  Row index lists use the same
delta + byte-plane + lzma scheme without the rounding.
"""
from __future__ import annotations

import lzma

import numpy as np

QBITS = 36
QUANT_ABS_ERR = 2.0 ** -(QBITS + 1)


def _pack_int(q: np.ndarray) -> bytes:
    d = np.diff(q.astype(np.int64).ravel(), prepend=np.int64(0))
    planes = d.view(np.uint8).reshape(-1, 8).T.copy()      # byte planes: high bytes compress away
    return lzma.compress(planes.tobytes(), preset=9)


def _unpack_int(blob: bytes, n: int) -> np.ndarray:
    planes = np.frombuffer(lzma.decompress(blob), np.uint8).reshape(8, n)
    d = planes.T.copy().view(np.int64).ravel()
    return np.cumsum(d)


def pack_field(T: np.ndarray) -> np.ndarray:
    """float64 array -> uint8 blob (shape kept by the caller)."""
    q = np.round(np.asarray(T, np.float64) * 2.0 ** QBITS).astype(np.int64)
    return np.frombuffer(_pack_int(q), np.uint8)


def unpack_field(blob: np.ndarray, n: int) -> np.ndarray:
    return _unpack_int(bytes(blob), n).astype(np.float64) * 2.0 ** -QBITS


def pack_rows(rows: np.ndarray) -> np.ndarray:
    return np.frombuffer(_pack_int(np.asarray(rows, np.int64)), np.uint8)


def unpack_rows(blob: np.ndarray, n: int) -> np.ndarray:
    return _unpack_int(bytes(blob), n)
