"""Lane model of a 'group' formulation of the density sweep (design tool, CPU only): G lanes per
home particle, 32/G particles per warp, lanes over CANDIDATES instead of one lane per particle.
Per direction the group's lanes split over the two sides (+d prefix, -d suffix of the reversed
lists), each lane evaluating two candidates per step (one FFMA2 pair, every candidate
interacted branch-free, no hit stacks), and a side stops after the step whose farthest entry
is outside the particle's window (or at the end of the neighbour's list); the self cell is
swept by all G lanes.  The warp runs the longest group per direction.  Reports issued
candidate slots per particle (G lanes x 2 per group step) next to the v5 figures of
scripts/sim_lanes.py.  usage: python scripts/sim_groups.py [c3|c5] [n_rowpairs]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import synth  # noqa: E402

GAMMA = synth.GAMMA
DIRS = [(0, 0, 1), (0, 1, -1), (0, 1, 0), (0, 1, 1)] + [(1, b, c) for b in (-1, 0, 1) for c in (-1, 0, 1)]


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    nrp = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    p = synth.make(cfg)
    nc = p.nc
    x = p.xyzh[:, :3].astype(np.float64)
    H = GAMMA * p.xyzh[:, 3].astype(np.float64)
    ijk = np.clip(np.floor(x * nc), 0, nc - 1).astype(np.int64)
    cid = (ijk[:, 0] * nc + ijk[:, 1]) * nc + ijk[:, 2]
    order = np.argsort(cid, kind="stable")
    start = np.searchsorted(cid[order], np.arange(nc ** 3 + 1))
    rng = np.random.default_rng(0)

    def cell(a, b, c):
        k = ((a % nc) * nc + (b % nc)) * nc + (c % nc)
        return order[start[k]:start[k + 1]]

    def side(i, ci, d, s):
        a, b, c = ci
        j = cell(a + s * d[0], b + s * d[1], c + s * d[2])
        ax = np.array(d, np.float64) / np.linalg.norm(d)
        dx = x[j] - x[i]
        dx -= np.round(dx)
        sep = dx @ ax * s
        return int(np.sum(sep < H[i])), len(j)

    Gs = (2, 4, 8)
    res = {g: 0 for g in Gs}
    cand = 0
    parts = 0
    for _ in range(nrp):
        xo, yp = rng.integers(0, nc), rng.integers(0, (nc + 1) // 2)
        seq = []
        for z in range(nc):
            for y in (2 * yp, 2 * yp + 1):
                if y < nc:
                    seq += [(i, (xo, y, z)) for i in cell(xo, y, z)]
        for t0 in range(0, len(seq) - 255, 256):
            tile = seq[t0:t0 + 256]
            W = np.zeros((256, 13, 2), np.int64)      # window length per side
            N = np.zeros((256, 13, 2), np.int64)      # neighbour cell count per side
            S = np.zeros(256, np.int64)
            for li, (i, ci) in enumerate(tile):
                for k, d in enumerate(DIRS):
                    for m, s in enumerate((1, -1)):
                        W[li, k, m], N[li, k, m] = side(i, ci, d, s)
                S[li] = len(cell(*ci)) - 1
            cand += W.sum() + S.sum()
            parts += 256
            for G in Gs:
                per = G                                       # candidates per side per step (G/2 lanes x 2)
                if G == 2:
                    per = 2                                   # one lane per side
                steps_side = np.where(W < N, W // per + 1, -(-W // per))
                steps_dir = steps_side.max(2)                 # (256, 13): both sides in lockstep
                self_steps = -(-S // (2 * G))
                P = 32 // G
                for w0 in range(0, 256, P):
                    sl = slice(w0, w0 + P)
                    res[G] += (steps_dir[sl].max(0).sum() + self_steps[sl].max()) * 2 * G * P
    print(f"{cfg}: {parts} particles; exact window candidates/particle {cand / parts:.1f} (self incl.)")
    for G in Gs:
        s = res[G] / parts
        red = 22 * np.log2(G) * 2 * 32 / (32 // G) / 1.0 if G > 1 else 0
        print(f"  G={G}: {s:6.1f} candidate slots/particle (efficiency {cand / parts / s:.3f}); "
              f"x ~32 instr = {s * 32:6.0f} lane-slots + reduction {red:5.0f}")


if __name__ == "__main__":
    main()
