"""CPU emulation of motion_fused_kernel's warp algorithm (32 lanes as numpy
vectors) -- a debugging aid that separates logic errors from codegen."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import oracle as O  # noqa: E402

R = 32
U = np.uint32


def W8(a, b, c, d):
    return U(a | (b << 8) | (c << 16) | (d << 24))


def dp4a(a, b, c):
    a = a.astype(np.uint64)
    r = c.astype(np.uint64) if isinstance(c, np.ndarray) else np.uint64(c)
    for i in range(4):
        r = r + ((a >> np.uint64(8 * i)) & np.uint64(0xFF)) * np.uint64((int(b) >> (8 * i)) & 0xFF)
    return (r & np.uint64(0xFFFFFFFF)).astype(U)


def byte(x, i):
    return (x >> U(8 * i)) & U(0xFF)


def prmt(a, b, s, sign=False):
    out = np.zeros_like(a)
    for k in range(4):
        sel = (s >> (4 * k)) & 0xF
        src = a if (sel & 7) < 4 else b
        v = byte(src, sel & 3)
        if sel & 8:
            v = np.where(v & U(0x80), U(0xFF), U(0))
        out |= v << U(8 * k)
    return out


def shfl_up(x):
    return np.concatenate([x[:1], x[:-1]])


def shfl_down(x):
    return np.concatenate([x[1:], x[-1:]])


def load_gray8(frame, y, xs, W, H):
    g0 = np.zeros(32, U)
    g1 = np.zeros(32, U)
    if y < 0 or y >= H:
        return g0, g1
    for l, x in enumerate(xs):
        px = [int(frame[y * W + x + i]) if 0 <= x + i < W else 0 for i in range(8)]
        g0[l] = W8(*px[:4])
        g1[l] = W8(*px[4:])
    return g0, g1


def hgauss4(L, C, Rw):
    h0 = dp4a(L, W8(0, 0, 1, 4), dp4a(C, W8(6, 4, 1, 0), 0))
    h1 = dp4a(L, W8(0, 0, 0, 1), dp4a(C, W8(4, 6, 4, 1), 0))
    h2 = dp4a(C, W8(1, 4, 6, 4), dp4a(Rw, W8(1, 0, 0, 0), 0))
    h3 = dp4a(C, W8(0, 1, 4, 6), dp4a(Rw, W8(4, 1, 0, 0), 0))
    return prmt(h0, h1, 0x5410), prmt(h2, h3, 0x5410)


def vgauss(a, b, c, d, e):
    A = a + e + U(0x00800080)
    B = b + d
    return c * U(6) + (B * U(4) + A)


def vabsdiff4(a, b):
    out = np.zeros_like(a)
    for i in range(4):
        x, y = byte(a, i).astype(np.int64), byte(b, i).astype(np.int64)
        out |= np.abs(x - y).astype(U) << U(8 * i)
    return out


def maj(a, b, c):
    return (a & b) | (a & c) | (b & c)


def sel(s, a, b):
    return (a & s) | (b & ~s)


def maj5(c, u, d, l, r):
    any3, m3, all3 = c | u | d, maj(c, u, d), c & u & d
    X = sel(r, any3, m3)
    Y = sel(r, m3, all3)
    return sel(l, X, Y)


def masks(xs, W):
    gm = np.zeros((2, 32), U)
    mm = np.zeros((2, 32), U)
    for l, x in enumerate(xs):
        for w in range(2):
            for i in range(4):
                xi = x + 4 * w + i
                if xi < 2 or xi >= W - 2:
                    gm[w, l] |= U(0xFF << (8 * i))
                if xi == 0 or xi == W - 1:
                    mm[w, l] |= U(0xFF << (8 * i))
    return gm, mm


def frame_pass(frame, out, prev_s, W, H, y0, xs, gm, mm, thr, mode):
    k = U((127 - thr) * 0x01010101) if thr <= 127 else U((255 - thr) * 0x01010101)
    tsel = U(0xFFFFFFFF) if thr <= 127 else U(0)
    slots = {}
    gy_begin, gy_end = y0 - 3, min(y0 + R + 3, H + 3)

    def produce(gy):
        g0, g1 = load_gray8(frame, gy, xs, W, H)
        left, right = shfl_up(g1), shfl_down(g0)
        h0, h1 = hgauss4(left, g0, g1)
        h2, h3 = hgauss4(g0, g1, right)
        slots[gy] = {"h": [h0, h1, h2, h3], "g": [g0, g1], "t": [None, None]}

    for gy in range(gy_begin, gy_begin + 4):
        produce(gy)
    for gy in range(gy_begin + 4, gy_end):
        produce(gy)
        gc = gy - 2
        if gc < y0 - 1 or gc > y0 + R:
            continue
        r4, r3, r2, r1, r0 = (slots[gy - 4], slots[gy - 3], slots[gy - 2], slots[gy - 1], slots[gy])
        gw = [None, None]
        if gc < 2 or gc >= H - 2:
            gw = list(r2["g"])
        else:
            for w in range(2):
                v0 = vgauss(*(s["h"][2 * w] for s in (r4, r3, r2, r1, r0)))
                v1 = vgauss(*(s["h"][2 * w + 1] for s in (r4, r3, r2, r1, r0)))
                gw[w] = sel(gm[w], r2["g"][w], prmt(v0, v1, 0x7531))
        idx = gc - (y0 - 1)
        if mode == 0:
            prev_s[idx] = np.stack(gw)
            continue
        pv = prev_s[idx].copy()
        prev_s[idx] = np.stack(gw)
        for w in range(2):
            d = vabsdiff4(gw[w], pv[w])
            t = (d & U(0x7F7F7F7F)) + k
            r2["t"][w] = maj(t, d, tsel)
        m = gc - 1
        if m < y0 or m >= y0 + R or m >= H:
            continue
        c0, c1 = r3["t"]
        lnb, rnb = shfl_up(c1), shfl_down(c0)
        if m == 0 or m == H - 1:
            o0, o1 = c0, c1
        else:
            l0 = ((c0 << U(8)) | (lnb >> U(24))) & U(0xFFFFFFFF)
            r0w = (c0 >> U(8)) | ((c1 << U(24)) & U(0xFFFFFFFF))
            l1 = ((c1 << U(8)) | (c0 >> U(24))) & U(0xFFFFFFFF)
            r1w = (c1 >> U(8)) | ((rnb << U(24)) & U(0xFFFFFFFF))
            o0 = sel(mm[0], c0, maj5(c0, r4["t"][0], r2["t"][0], l0, r0w))
            o1 = sel(mm[1], c1, maj5(c1, r4["t"][1], r2["t"][1], l1, r1w))
        o0, o1 = prmt(o0, o0 * 0, 0xBA98), prmt(o1, o1 * 0, 0xBA98)
        for l, x in enumerate(xs):
            if 1 <= l <= 30:
                for i in range(8):
                    if 0 <= x + i < W:
                        word = o0[l] if i < 4 else o1[l]
                        out[m * W + x + i] = (int(word) >> (8 * (i & 3))) & 0xFF


def run(frames, W, H, thr=32, chunk=None):
    n = frames.size // (W * H)
    out = np.zeros(n * W * H, np.uint8)
    tiles = (W + 239) // 240
    bands = (H + R - 1) // R
    chunk = chunk or n
    for tx in range(tiles):
        xs = [tx * 240 - 8 + 8 * l for l in range(32)]
        gm, mm = masks(xs, W)
        for b in range(bands):
            y0 = b * R
            for f0 in range(0, n, chunk):
                prev_s = np.zeros((R + 2, 2, 32), U)
                if f0 > 0:
                    frame_pass(frames[(f0 - 1) * W * H:f0 * W * H], None, prev_s, W, H, y0, xs, gm, mm, thr, 0)
                for f in range(f0, min(f0 + chunk, n)):
                    frame_pass(frames[f * W * H:(f + 1) * W * H], out[f * W * H:(f + 1) * W * H], prev_s,
                               W, H, y0, xs, gm, mm, thr, 1)
    return out


if __name__ == "__main__":
    for (w, h, n, chunk) in [(16, 8, 2, 1), (96, 40, 1, None), (33, 29, 3, 1)]:
        f = O.synth_bytes(n * w * h, 606)
        got = run(f, w, h, 32, chunk)
        want = O.motion_gray(f, w, h)
        bad = np.nonzero(got != want)[0]
        print(w, h, n, chunk, "bad", bad.size, "first", [(int(i) // (w * h), int(i) % (w * h) // w, int(i) % w) for i in bad[:5]])
