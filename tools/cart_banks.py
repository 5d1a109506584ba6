"""Offline search behind the shared-memory layout of the tensor-product
Cartesian kernel (paper_1711_03590_b200/csrc/sipg_cart.cuh, cart_pad):
for every k = 2..11 and word size (8-byte words: 16 banks per half-warp
request; 4-byte words: 32 banks per warp request), the plane-stride padding
S2 = k^2 + pad (row stride k) for which the bank residues of the first entries
of the x-lines (k i + S2 j) and of the y-lines (i + S2 j) are spread most
evenly, i.e. for which a permutation of the lines over the threads exists with
residue(thread t) = (t + beta) mod #banks for all but a few lines. The z-lines
(i + k j = t) need no permutation. The host builds the permutations with the
same greedy matching (sipg_launch.cuh, cart_perm_host).

usage: python tools/cart_banks.py      -> the two pad tables and the unmatched-line counts
"""


def residues(K, S2, axis, nb):
    """bank residue of line p = i + K j (first entry) along x (axis 0) or y (axis 1)"""
    return [((K * i + S2 * j) if axis == 0 else (i + S2 * j)) % nb for j in range(K) for i in range(K)]


def unmatched(K, S2, axis, nb):
    """lines that do not fit the run (t + beta) mod nb, for the best beta"""
    res = residues(K, S2, axis, nb)
    have = [0] * nb
    for r in res:
        have[r] += 1
    best = None
    for beta in range(nb):
        need = [0] * nb
        for t in range(K * K):
            need[(t + beta) % nb] += 1
        bad = sum(max(0, need[r] - have[r]) for r in range(nb))
        if best is None or bad < best[0]:
            best = (bad, beta)
    return best


def main():
    for nb, name in ((16, "8-byte words"), (32, "4-byte words")):
        pads = []
        for K in range(2, 12):
            best = None
            for pad in range(0, 9):
                S2 = K * K + pad
                u = [unmatched(K, S2, a, nb) for a in (0, 1)]
                key = (u[0][0] + u[1][0], pad)
                if best is None or key < best[0]:
                    best = (key, pad, u)
            pads.append(best[1])
            print(f"{name}: k={K} pad={best[1]} unmatched lines x/y: {best[2][0][0]}/{best[2][1][0]} of {K * K}")
        print(f"{name}: cart_pad table (k = 2..11) = {pads}")


if __name__ == "__main__":
    main()
