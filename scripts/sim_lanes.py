"""Lane-efficiency model of the density sweep (design tool, CPU only).

For a sample of home cells of a config, computes every home particle's exact window length
per direction segment (+d prefix, -d suffix, as the kernel's bisection does, fp64 here),
forms warps the way k_v4_tiles/k_density_v5 do (256-particle runs of a row pair, slice by
slice, 32 consecutive particles per warp) and reports the issued slots per particle of
alternative sweep organisations:
  per_dir   : trip per direction = max over the warp's lanes of (len+ + len-)   (v5)
  per_pair  : directions swept in pairs (v4)
  cursor    : one stream over all 13 directions per lane (max over lanes of the total)
and the hit-drain efficiency.
usage: python scripts/sim_lanes.py [c3|c5] [n_rowpairs]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import synth  # noqa: E402

GAMMA = synth.GAMMA
DIRS = [(0, 0, 1), (0, 1, -1), (0, 1, 0), (0, 1, 1)] + [(1, b, c) for b in (-1, 0, 1) for c in (-1, 0, 1)]


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    nrp = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    p = synth.make(cfg)
    nc = p.nc
    x = p.xyzh[:, :3].astype(np.float64)
    H = GAMMA * p.xyzh[:, 3].astype(np.float64)
    ijk = np.clip(np.floor(x * nc), 0, nc - 1).astype(np.int64)
    cid = (ijk[:, 0] * nc + ijk[:, 1]) * nc + ijk[:, 2]
    order = np.argsort(cid, kind="stable")
    start = np.searchsorted(cid[order], np.arange(nc ** 3 + 1))
    cl = 1.0 / nc
    rng = np.random.default_rng(0)

    def cell(a, b, c):
        k = ((a % nc) * nc + (b % nc)) * nc + (c % nc)
        return order[start[k]:start[k + 1]]

    def wlen(i, ci, d, s):
        """window length of particle i in neighbour cell ci + s d."""
        a, b, c = ci
        j = cell(a + s * d[0], b + s * d[1], c + s * d[2])
        dv = np.array(d, np.float64)
        ax = dv / np.linalg.norm(dv)
        dx = x[j] - x[i]
        dx -= np.round(dx)                            # minimum image
        sep = dx @ ax * s
        return int(np.sum(sep < H[i]))

    res = {"per_dir": 0, "per_pair": 0, "cursor": 0, "self": 0, "cand": 0, "parts": 0}
    for _ in range(nrp):
        xo, yp = rng.integers(0, nc), rng.integers(0, (nc + 1) // 2)
        seq = []
        for z in range(nc):
            for y in (2 * yp, 2 * yp + 1):
                if y >= nc:
                    continue
                for i in cell(xo, y, z):
                    seq.append((i, (xo, y, z)))
        for t0 in range(0, len(seq) - 255, 256):    # full tiles of 256
            tile = seq[t0:t0 + 256]
            LT = np.zeros((256, 13), np.int64)
            ST = np.zeros(256, np.int64)
            for li, (i, ci) in enumerate(tile):
                for k, d in enumerate(DIRS):
                    LT[li, k] = wlen(i, ci, d, 1) + wlen(i, ci, d, -1)
                ST[li] = len(cell(*ci)) - 1
            orders = {"seq": np.arange(256), "byH": np.argsort(-H[[i for i, _ in tile]], kind="stable"),
                      "bytotal": np.argsort(-(LT.sum(1) + ST), kind="stable")}
            for name, o in orders.items():
                for w in range(8):
                    sel = o[32 * w:32 * w + 32]
                    L, nself = LT[sel], ST[sel]
                    pad = lambda a, q: ((a + q - 1) // q) * q          # noqa: E731
                    for key, val in (("per_dir", L.max(0).sum()), ("per_dir_r8", pad(L.max(0), 8).sum()),
                                     ("per_dir_r4", pad(L.max(0), 4).sum()),
                                     ("cursor_p2", (pad(L, 2).sum(1) + pad(nself + 1, 2)).max()),
                                     ("cursor_p4", (pad(L, 4).sum(1) + pad(nself + 1, 4)).max()),
                                     ("per_pair", sum(L[:, k:k + 2].sum(1).max() for k in range(0, 13, 2))),
                                     ("cursor", L.sum(1).max()), ("cursor_all", (L.sum(1) + nself).max()),
                                     ("self", nself.max() + 1)):
                        res.setdefault(name + key, 0)
                        res[name + key] += val * 32
            res["cand"] += LT.sum() + ST.sum()
            res["parts"] += 256
    n = res["parts"]
    print(f"{cfg}: {n} particles; window candidates/particle {res['cand'] / n:.1f} (self incl.)")
    for o in ("seq", "byH", "bytotal"):
        for k in ("per_dir", "per_pair", "cursor"):
            s = res[o + k] / n
            print(f"  {o:8s} {k:9s} neighbour slots/particle {s:7.1f}   self {res[o + 'self'] / n:5.1f}   "
                  f"efficiency {res['cand'] / (res[o + k] + res[o + 'self']):.3f}")
        print(f"  {o:8s} cursor incl. self: {res[o + 'cursor_all'] / n:7.1f}  efficiency "
              f"{res['cand'] / res[o + 'cursor_all']:.3f}")
        sl = res[o + 'self'] / n
        for k, c in (("per_dir_r8", 11), ("per_dir_r4", 11.5), ("cursor_p2", 14), ("cursor_p4", 12.5)):
            slots = res[o + k] / n + (sl if k.startswith("per") else 0)
            print(f"  {o:8s} {k:10s} slots/particle {slots:7.1f}  x {c} instr = {slots * c:7.0f} lane-slots")


if __name__ == "__main__":
    main()
