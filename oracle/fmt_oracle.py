"""CPU restatement of the reference's matches-file writer.

TEST INFRASTRUCTURE ONLY: imported by tests/ as the checker of the GPU
formatter (paper_2312_01476_b200/csrc/sjb_fmt.cu); the product never imports
it.

The reference (cli.py:99-108) writes one line per match,
``f"{left},{right},{_fmt_sim(sim)}\\n"`` with
``_fmt_sim(v) = numpy.format_float_positional(numpy.float32(v), unique=True,
trim="-")``.  The float formatting is third-party code: numpy's Dragon4
(numpy >= 1.14; 2.3.5 here), shortest-unique digit generation.  Its
published algorithm (Steele & White free-format printing with Juckett's
margins) is restated below in exact Python integers, and pinned against
numpy itself by tests/test_oracle.py (whole strided binades, random bit
patterns, every power of two +-1 ulp): numpy treats the rounding-interval
boundaries as inclusive when the mantissa is even, and the strict variant
measurably differs (e.g. 0x4F13C45E -> "2479120000", not "2479119900").

``matches_file_reference`` is the reference writer itself (numpy per line),
the oracle the GPU output is compared with byte for byte.
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np

_LOG10_2 = 0.30102999566398119521373889472449


def shortest_digits(bits: int) -> Tuple[str, int]:
    """Shortest-unique digits of a positive finite nonzero float32 given by its
    bit pattern, and the decimal exponent of the first digit."""
    be, f = (bits >> 23) & 0xFF, bits & 0x7FFFFF
    if be:
        m, ex, mbit = f | (1 << 23), be - 150, 23
        unequal = f == 0 and be != 1     # power of two: the lower gap is half
    else:
        m, ex, mbit = f, -149, f.bit_length() - 1
        unequal = False
    if unequal:
        if ex > 0:
            val, scale, ml, mh = (4 * m) << ex, 4, 1 << ex, 1 << (ex + 1)
        else:
            val, scale, ml, mh = 4 * m, 1 << (-ex + 2), 1, 2
    else:
        if ex > 0:
            val, scale, ml = (2 * m) << ex, 2, 1 << ex
        else:
            val, scale, ml = 2 * m, 1 << (-ex + 1), 1
        mh = ml
    de = math.ceil((mbit + ex) * _LOG10_2 - 0.69)   # first-digit exponent, maybe 1 low
    if de > 0:
        scale *= 10 ** de
    elif de < 0:
        p = 10 ** (-de)
        val, ml = val * p, ml * p
        mh = 2 * ml if unequal else ml
    if val >= scale:
        de += 1
    else:
        val, ml = val * 10, ml * 10
        mh = 2 * ml if unequal else ml
    exp10 = de - 1
    incl = (m & 1) == 0
    digits = []
    while True:
        d, val = divmod(val, scale)
        low = val <= ml if incl else val < ml
        high = val + mh >= scale if incl else val + mh > scale
        if low or high:
            break
        digits.append(d)
        val, ml = val * 10, ml * 10
        mh = 2 * ml if unequal else ml
    round_down = low
    if low == high:
        round_down = 2 * val < scale or (2 * val == scale and d % 2 == 0)
    if round_down:
        digits.append(d)
    elif d < 9:
        digits.append(d + 1)
    else:
        while digits and digits[-1] == 9:
            digits.pop()
        if digits:
            digits[-1] += 1
        else:
            digits, exp10 = [1], exp10 + 1
    return "".join(map(str, digits)), exp10


def fmt_sim(value) -> str:
    """Restated _fmt_sim (cli.py:99-102)."""
    bits = int(np.float32(value).view(np.uint32))
    sign = "-" if bits >> 31 else ""
    bits &= 0x7FFFFFFF
    if bits == 0:
        return sign + "0"
    if bits >= 0x7F800000:
        return "nan" if bits > 0x7F800000 else sign + "inf"
    ds, e = shortest_digits(bits)
    if e >= 0:
        body = ds + "0" * (e + 1 - len(ds)) if len(ds) <= e + 1 else ds[:e + 1] + "." + ds[e + 1:]
    else:
        body = "0." + "0" * (-e - 1) + ds
    return sign + body


def fmt_sim_numpy(value) -> str:
    """The reference's _fmt_sim verbatim in behaviour (cli.py:99-102)."""
    return np.format_float_positional(np.float32(value), unique=True, trim="-")


def matches_file_reference(lefts, rights, sims) -> bytes:
    """The reference writer's bytes (cli.py:105-108; MatchSet.__iter__
    yields int, int, float, core.py:137-139)."""
    out = []
    for l, r, s in zip(lefts, rights, sims):
        out.append(f"{int(l)},{int(r)},{fmt_sim_numpy(float(s))}\n")
    return "".join(out).encode("utf-8")


def probe_bits(n_random: int, seed: int = 0, stride: int = 97) -> np.ndarray:
    """float32 bit patterns that exercise the formatter: a strided sweep of
    [0.5, 1) and [1, 2), every power of two and its neighbours, denormals,
    extremes, and random finite patterns of both signs."""
    rng = np.random.default_rng(seed)
    parts = [np.arange(0x3F000000, 0x40000000, stride, dtype=np.uint64)]
    k = np.arange(1, 255, dtype=np.uint64) << np.uint64(23)
    parts += [k, k + 1, k - 1]
    parts.append(np.array([1, 2, 3, 0x7FFFFF, 0x800000, 0x7F7FFFFF, 0x3F800000, 0x3DCCCCCD,
                           0x4B800000, 0x4F13C45E, 0x3F7FFFFF, 0x33800000], dtype=np.uint64))
    parts.append(rng.integers(0, 0x7F800000, n_random, dtype=np.uint64))
    b = np.concatenate(parts).astype(np.uint32)
    sign = rng.integers(0, 2, b.size, dtype=np.uint32) << np.uint32(31)
    return np.concatenate([b, b[: b.size // 4] | sign[: b.size // 4]])
