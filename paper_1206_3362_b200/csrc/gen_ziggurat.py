"""Generate fwbf_ziggurat.h: the constants of numpy's standard-normal sampler.

The reference draws channel noise with numpy's `Generator(Philox).standard_normal`
(channel.py:36,49).  numpy (2.x, here 2.3.5) implements the 256-level
Marsaglia-Tsang ziggurat on 64-bit draws: idx = r & 0xff, a sign bit, a 52-bit
magnitude `rabs`; x = rabs * w[idx]; accept if rabs < k[idx]; otherwise the
base strip samples the tail beyond R by -log1p(-U)/R, and the other strips do
the wedge test f[idx] + (f[idx-1] - f[idx]) U < exp(-x^2/2).

numpy's C tables are not in this container (only .pxd stubs), so the
constants are PINNED BY MEASUREMENT, black-box, against the installed numpy:
  * w[i] (the only table that enters outputs directly) is the unique double
    with fl(rabs * w[i]) == |x| for every sampled first draw with that idx;
  * x_i = w[i] * 2^52; k[i] = uint64(x_{i-1} / x_i * 2^52) (k[0] = R / x_0,
    k[1] = 0); f[i] = exp(-x_i^2 / 2), f[0] = 1; these only decide rare
    accept/reject comparisons;
  * the full restatement is then replayed against numpy on 200 frames x 1023
    normals and must agree bit for bit (including tail and wedge events).

Run once in the build container:  python paper_1206_3362_b200/csrc/gen_ziggurat.py
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

R = 3.6541528853610088          # right-most ziggurat edge used by numpy
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "fwbf_ziggurat.h")

MASK = (1 << 64) - 1
PM0, PM1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
PW0, PW1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B


def philox4x64(ctr, key):
    """Philox4x64-10 (Salmon et al., SC'11) -- the bit generator of channel.py:49."""
    c, k = list(ctr), list(key)
    for _ in range(10):
        p0, p1 = PM0 * c[0], PM1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k[0], p1 & MASK, (p0 >> 64) ^ c[3] ^ k[1], p0 & MASK]
        k = [(k[0] + PW0) & MASK, (k[1] + PW1) & MASK]
    return c


class Stream:
    """numpy Philox(key=seed, counter=frame<<128): counter incremented before use."""

    def __init__(self, seed, frame):
        self.ctr = [0, 0, frame & MASK, (frame >> 64) & MASK]
        self.key = [seed & MASK, (seed >> 64) & MASK]
        self.buf = []

    def u64(self):
        if not self.buf:
            c = self.ctr
            for i in range(4):
                c[i] = (c[i] + 1) & MASK
                if c[i]:
                    break
            self.buf = philox4x64(c, self.key)[::-1]
        return self.buf.pop()

    def dbl(self):
        return (self.u64() >> 11) * (1.0 / 9007199254740992.0)


def pin_w(samples=400000, seed=11):
    raw = np.empty(samples, np.uint64)
    xs = np.empty(samples)
    for i in range(samples):
        raw[i] = np.random.Philox(key=seed, counter=i << 128).random_raw()
        xs[i] = np.random.Generator(np.random.Philox(key=seed, counter=i << 128)).standard_normal()
    idx = (raw & np.uint64(0xFF)).astype(np.int64)
    rabs = ((raw >> np.uint64(9)) & np.uint64(0x000FFFFFFFFFFFFF)).astype(np.float64)
    a = np.abs(xs)
    w = np.zeros(256)
    for k in range(256):
        sel = idx == k
        ratio = a[sel] / rabs[sel]
        med = np.median(ratio)
        cands = np.unique(ratio[np.abs(ratio / med - 1) < 1e-9])
        best = (-1, 0.0)
        for c in cands[:200]:
            for d in (-2, -1, 0, 1, 2):
                t = c
                for _ in range(abs(d)):
                    t = np.nextafter(t, np.inf if d > 0 else -np.inf)
                hits = int((rabs[sel] * t == a[sel]).sum())
                if hits > best[0]:
                    best = (hits, t)
        if best[0] < 0.5 * sel.sum():
            raise RuntimeError(f"could not pin w[{k}]")
        w[k] = best[1]
    return w


def tables(w):
    x = w * 2.0 ** 52
    k = [0] * 256
    k[0] = int(np.uint64(R / x[0] * 2.0 ** 52))
    for i in range(2, 256):
        k[i] = int(np.uint64(x[i - 1] / x[i] * 2.0 ** 52))
    f = [1.0] + [math.exp(-0.5 * x[i] * x[i]) for i in range(1, 256)]
    return k, f


def normal(s, w, k, f):
    inv_r = 1.0 / R
    while True:
        r = s.u64()
        idx = r & 0xFF
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * w[idx]
        if sign:
            x = -x
        if rabs < k[idx]:
            return x
        if idx == 0:
            while True:
                xx = -inv_r * math.log1p(-s.dbl())
                yy = -math.log1p(-s.dbl())
                if yy + yy > xx * xx:
                    return -(R + xx) if (rabs >> 8) & 1 else R + xx
        elif (f[idx - 1] - f[idx]) * s.dbl() + f[idx] < math.exp(-0.5 * x * x):
            return x


def main():
    w = pin_w()
    k, f = tables(w)
    for frame in range(200):
        s = Stream(3, frame)
        mine = np.array([normal(s, w, k, f) for _ in range(1023)])
        ref = np.random.Generator(np.random.Philox(key=3, counter=frame << 128)).standard_normal(1023)
        if not np.array_equal(mine, ref):
            raise RuntimeError(f"replay mismatch in frame {frame}")
    with open(OUT, "w") as fh:
        fh.write("// Generated by gen_ziggurat.py from numpy %s (black-box pinned); do not edit.\n"
                 % np.__version__)
        fh.write("#pragma once\n")
        fh.write("#define FWBF_ZIG_R %s\n" % float(R).hex())
        fh.write("#define FWBF_ZIG_W_INIT {%s}\n" % ", ".join(float(v).hex() for v in w))
        fh.write("#define FWBF_ZIG_K_INIT {%s}\n" % ", ".join("0x%016xull" % v for v in k))
        fh.write("#define FWBF_ZIG_F_INIT {%s}\n" % ", ".join(float(v).hex() for v in f))
    print("wrote", OUT)


if __name__ == "__main__":
    sys.exit(main())
