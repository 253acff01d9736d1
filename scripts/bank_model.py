"""Shared-memory bank model for the element kernel's node layouts (3D).

A warp-wide 64-bit shared load is served per half-warp; a half-warp needs as
many wavefronts as the largest number of distinct 8-byte words falling into
one of the 16 bank pairs. Optimal = 2 wavefronts per warp. The access pattern
of the volume passes: lane = one 1D line (one thread per line), all lanes of
a warp at the same line position; the staging/epilogue patterns (consecutive
nodes) are conflict-free for every layout below.

    python scripts/bank_model.py      -> mean / max wavefronts per warp load
"""


def lines_pattern(p1, padf, epb_lanes):
    d = 3
    lines = p1 ** (d - 1)
    res = []
    for n in range(d):
        s = p1 ** (d - 1 - n)
        for w0 in range(0, max(lines, 32), 32):
            for pos in range(p1):
                addrs = []
                for lane in range(32):
                    g = w0 + lane
                    el, m = divmod(g, lines) if epb_lanes else (0, g % lines)
                    node = (m // s) * p1 * s + m % s + pos * s
                    addrs.append(el * (p1 ** 3 + 64) + padf(node))
                tot = 0
                for half in (addrs[:16], addrs[16:]):
                    banks = {}
                    for a in set(half):
                        banks.setdefault(a % 16, set()).add(a)
                    tot += max(len(v) for v in banks.values())
                res.append(tot)
    return sum(res) / len(res), max(res)


if __name__ == "__main__":
    for p1, name, f in [
        (4, "pad (node + node/4)", lambda x: x + x // 4),
        (4, "swizzle node ^ 5(node>>4)", lambda x: x ^ (((x >> 4) * 5) & 15)),
        (8, "pad (node + node/8)", lambda x: x + x // 8),
        (8, "swizzle node ^ (node>>3)", lambda x: x ^ ((x >> 3) & 15)),
    ]:
        print("p+1=%d %-28s mean %.2f max %d wavefronts per warp load" % ((p1, name) + lines_pattern(p1, f, True)))
