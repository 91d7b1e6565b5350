"""DMMA work per point of the tensor-core gather for box shapes bx x by x 8
at Poisson point density rho per cell (m = 6): units are a box's points
sorted by depth in chunks of 8, each costing (row slots / 8) * KC * 2 + 24
DMMAs with KC = max(4, ceil((span + 13) / 4)) and the row schedule of
vfn_gather_tc.cu (8-row tiles per x, then x pairs / quads / octets).
Prints DMMA per point (mean points per unit).  Usage: python tools/box_shape_sim.py"""
import numpy as np

rng = np.random.default_rng(0)


def slots(XB, YB):
    y8 = YB // 8
    r = YB - 8 * y8
    r4 = r >= 4
    r -= 4 * r4
    r2 = r >= 2
    r -= 2 * r2
    return 8 * (y8 * XB + r4 * ((XB + 1) // 2) + r2 * ((XB + 3) // 4) + r * ((XB + 7) // 8))


def sim(rho, bx, by, tz=8, m=6, nbox=20000):
    W = 2 * m + 1
    S = slots(bx + 2 * m, by + 2 * m)
    tot = pts = units = 0
    for c in rng.poisson(rho * bx * by * tz, nbox):
        if c == 0:
            continue
        d = np.sort(rng.integers(0, tz, c))
        for i in range(0, c, 8):
            span = d[i:i + 8][-1] - d[i]
            kc = max((W + 3) // 4, -(-(span + W) // 4))
            tot += S // 8 * kc * 2 + 24
            units += 1
        pts += c
    return tot / pts, pts / units


for rho in (0.12, 0.24, 0.48, 1.0, 2.0, 4.0):
    print(rho, " ".join("%dx%d:%.1f(%.1f)" % (bx, by, *sim(rho, bx, by))
                        for bx, by in ((1, 1), (1, 2), (2, 1), (2, 2), (2, 4), (4, 4))))
