"""Geometric census of the R4 full events (numpy, no GPU): how many of a
full event's point pairs lie in the mollifier shell, and how many shell
polynomial evaluations per lane different vote / compaction schemes need.

R4: h = 1/64, delta = 0.1, eps = h/2, GL3 points, L_max = 2 sub-cells of
the outer element against an inner element at every cell offset within the
stencil (interior, unweighted).  A "full" event has point pairs on both
sides of the shell boundaries.  Lanes = the 27 inner points (k_hex).

    python tools/shell_census.py
"""

import itertools

import numpy as np


def main():
    h = 1 / 64
    delta, eps = 0.1, h / 2
    dm2, dp2 = (delta - eps) ** 2, (delta + eps) ** 2
    g = np.sqrt(3 / 5)
    t = np.array([(1 - g) / 2, 0.5, (1 + g) / 2])
    R = 7
    Y = np.array([[t[i] * h, t[j] * h, t[k] * h] for k in range(3)
                  for j in range(3) for i in range(3)])
    frac, line, point, ideal, per_x = [], [], [], [], []
    for d in itertools.product(range(-R, R + 1), repeat=3):
        lo = np.array(d) * h
        for sub in itertools.product((0, 1), repeat=3):
            slo = lo + np.array(sub) * h / 2
            X = np.array([[slo[0] + t[a] * h / 2, slo[1] + t[b] * h / 2,
                           slo[2] + t[c] * h / 2] for a in range(3)
                          for b in range(3) for c in range(3)])
            D2 = ((X[None] - Y[:, None]) ** 2).sum(-1)
            if (D2 >= dp2).all() or (D2 < dm2).all():
                continue
            sh = (D2 >= dm2) & (D2 < dp2)
            s4 = sh.reshape(27, 3, 3, 3)
            frac.append(sh.mean())
            line.append(3 * s4.any(axis=(0, 3)).sum())
            point.append(s4.any(axis=0).sum())
            ideal.append(np.ceil(sh.sum() / 32))
            per_x.append(sum(np.ceil(s4[:, a].sum() / 32) for a in range(3)))
    print(f"full events: {len(frac)}; shell share of their point pairs "
          f"{np.mean(frac):.3f}")
    print("shell polynomial evaluations per lane and event:")
    print(f"  vote per (a, b) z-line (3 points) {np.mean(line):.1f}")
    print(f"  vote per point                    {np.mean(point):.1f}")
    print(f"  compaction per x node (32/round)  {np.mean(per_x):.1f}")
    print(f"  ideal compaction per event        {np.mean(ideal):.1f}")
    print("  no vote                           27")


if __name__ == "__main__":
    main()
