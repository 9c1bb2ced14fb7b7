"""Conversions between the two domain encodings used at the parity boundary.

* "member": flat uint8[R], R = sum(d); byte rowbase[i] + (v - lo_i) is 1 iff v in
  dom(x_i).  This is the oracle's encoding (plain, one byte per value).
* "bitmap": the C-ABI encoding (include/ct.h): uint64 words, each variable owns a
  word-aligned run of ceil(d_i/64) words starting at dom_word_offsets(d)[i];
  value v of x_i is bit (v - lo_i) % 64 of word off_i + (v - lo_i) // 64,
  LSB-first.  Bits >= d_i are zero.

Pure data layout: no GAC arithmetic here.
"""
from __future__ import annotations

import numpy as np


def dom_word_offsets(d) -> np.ndarray:
    d = np.asarray(d, dtype=np.int64)
    words = (d + 63) // 64
    return np.concatenate([[0], np.cumsum(words)]).astype(np.int64)


def row_bases(d) -> np.ndarray:
    d = np.asarray(d, dtype=np.int64)
    return np.concatenate([[0], np.cumsum(d)]).astype(np.int64)


def full_member(d) -> np.ndarray:
    return np.ones(int(np.sum(d)), dtype=np.uint8)


def member_to_bitmap(member: np.ndarray, d) -> np.ndarray:
    d = np.asarray(d, dtype=np.int64)
    offs = dom_word_offsets(d)
    rb = row_bases(d)
    out = np.zeros(int(offs[-1]), dtype=np.uint64)
    for i in range(d.size):
        m = np.asarray(member[rb[i]:rb[i + 1]], dtype=np.uint8)
        nw = int(offs[i + 1] - offs[i])
        padded = np.zeros(nw * 64, dtype=np.uint8)
        padded[: m.size] = m
        bits = np.packbits(padded.reshape(nw, 64), axis=1, bitorder="little")  # [nw][8] bytes
        out[offs[i]:offs[i + 1]] = bits.view("<u8").reshape(nw)
    return out


def bitmap_to_member(bitmap: np.ndarray, d) -> np.ndarray:
    d = np.asarray(d, dtype=np.int64)
    offs = dom_word_offsets(d)
    rb = row_bases(d)
    out = np.zeros(int(rb[-1]), dtype=np.uint8)
    bm = np.ascontiguousarray(np.asarray(bitmap, dtype=np.uint64))
    for i in range(d.size):
        words = bm[offs[i]:offs[i + 1]]
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")
        out[rb[i]:rb[i + 1]] = bits[: d[i]]
    return out


def bitmaps_to_members(bitmaps: np.ndarray, d) -> np.ndarray:
    """[S][Wd] -> [S][R]"""
    return np.stack([bitmap_to_member(b, d) for b in bitmaps]) if len(bitmaps) else np.zeros((0, int(np.sum(d))), np.uint8)


def bits_to_bool(words: np.ndarray, nbits: int) -> np.ndarray:
    """uint64 words (LSB-first) -> uint8[nbits] (tuple j -> word j//64, bit j%64)."""
    b = np.unpackbits(np.ascontiguousarray(words, dtype=np.uint64).view(np.uint8), bitorder="little")
    return b[:nbits]
