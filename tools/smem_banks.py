"""Shared-memory bank-conflict model of the fused SIPG apply kernel's access
patterns (sipg_kernel.cuh / sipg_faces.cuh), used to choose the padded
strides. 64-bit accesses: a warp request is served per half-warp; within a
half-warp, 8-byte words that map to the same bank pair ((addr/8) % 16) but
differ serialize (identical words broadcast). Prints wavefronts per warp
request relative to the ideal (2 for a full warp).

usage: python tools/smem_banks.py [K] [S1] [S2pad] [cellpad]
"""
import sys
from collections import defaultdict


def wavefronts(addrs):
    """addrs: list of (thread, word address or None) for one warp."""
    total = 0
    for half in (0, 1):
        banks = defaultdict(set)
        for t, a in addrs:
            if a is None or (t % 32) // 16 != half:
                continue
            banks[a % 16].add(a)
        total += max((len(v) for v in banks.values()), default=0)
    return total


def model(K, S1, S2, FK, cell, NC, P):
    FS = S2 * K
    FP = FK * K
    NL = P // K
    THREADS = NC * P
    pats = {}

    def warp_sum(fn):
        w = ideal = 0
        for w0 in range(0, THREADS, 32):
            addrs = []
            for t in range(w0, min(w0 + 32, THREADS)):
                lc, p = divmod(t, P)
                a = fn(lc, p)
                addrs.append((t, None if a is None else lc * cell + a))
            n = sum(1 for _, a in addrs if a is not None)
            if n == 0:
                continue
            w += wavefronts(addrs)
            ideal += 2 if n > 16 else 1
        return w / ideal

    for ax in range(3):
        def pid(p, m, ax=ax):
            if ax == 0:
                return m + S1 * (p % K) + S2 * (p // K)
            if ax == 1:
                return (p % K) + S1 * m + S2 * (p // K)
            return (p % K) + S1 * (p // K) + S2 * m
        pats[f"pencil{ax}"] = max(warp_sum(lambda lc, p, m=m: pid(p, m)) for m in range(K))
    fpt = lambda p: (p % K) + FK * (p // K)
    pats["facept"] = warp_sum(lambda lc, p: fpt(p))
    for T in (0, 1):
        def line(lc, p, m, T=T):
            # for (t = p; t < 4 NL; t += P): f = t / NL, l = t % NL (first trip)
            f, l = divmod(p, NL)
            if f >= 4:
                return None
            base = f * FP
            return base + (m + FK * l if T == 0 else l + FK * m)
        pats[f"line{T}"] = max(warp_sum(lambda lc, p, m=m: line(lc, p, m)) for m in range(K))
    return pats


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    P = K * K
    NC = max(1, 192 // P)
    for S1 in sorted({K, K + 1, K + 2, K + 3}):
        for pad2 in (0, 1, 2, 3):
            S2 = S1 * K + pad2
            for FK in sorted({K, K + 1, S1}):
                base = (4 * S2 * K) + 20 * FK * K + 12
                for cpad in (0, 2, 4, 6, 8, 10, 12, 14):
                    cell = base + cpad
                    pats = model(K, S1, S2, FK, cell, NC, P)
                    score = (2 * pats["pencil0"] + 2 * pats["pencil1"] + 2 * pats["pencil2"]
                             + pats["facept"] + pats["line0"] + pats["line1"]) / 9
                    print(f"S1={S1} S2={S2} FK={FK} cell={cell}: score {score:.3f} " +
                          " ".join(f"{k}={v:.2f}" for k, v in pats.items()))


if __name__ == "__main__":
    main()
