"""CPU simulation of the row grouping on the largest cfg3 element: kept pairs under the
centre/radius bound with tiles as built, split at far chain transitions, or split at
every seed group (dev tool; uses the oracle cover/membership)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2011_03209_b200 import workloads
from oracle import mapper_oracle as O
w = workloads.CONFIGS["cfg3"]
X = workloads.points(w)
F = np.sqrt((X * X).sum(1))
axes = [O.cover_axis(F, 40, 0.3)]
members = O.membership(F[:, None], axes)
sizes = [len(m) for m in members]
k = int(np.argsort(sizes)[-5])  # a large element
rows = members[k]; P = X[rows]; n = len(rows)
print("element", k, "n", n, flush=True)
S = 64
seeds = P[(np.arange(S) * n) // S]
# chain order over first 32 dims (greedy NN from seed 0)
sd = seeds[:, :32].astype(np.float32)
D = ((sd[:, None, :] - sd[None, :, :]) ** 2).sum(-1)
used = np.zeros(S, bool); cur = 0; used[0] = True; order = [0]
for _ in range(S - 1):
    dd = np.where(used, np.inf, D[cur]); cur = int(np.argmin(dd)); used[cur] = True; order.append(cur)
rank = np.empty(S, int); rank[order] = np.arange(S)
# assignment (first 32 dims)
x32 = P[:, :32].astype(np.float32)
sc = (sd * sd).sum(1)[None, :] - 2 * x32 @ sd.T
g = np.argmin(sc, 1)
key = rank[g]
perm = np.argsort(key, kind="stable")
eps = w.eps
def kept_pairs(tiles):
    C = np.array([P[t].mean(0) for t in tiles]); R = np.array([np.sqrt(((P[t] - C[i]) ** 2).sum(1)).max() for i, t in enumerate(tiles)])
    Dc = np.sqrt(((C[:, None, :] - C[None, :, :]) ** 2).sum(-1))
    keep = (Dc - (R[:, None] + R[None, :])) <= eps
    iu = np.triu_indices(len(tiles))
    sz = np.array([len(t) for t in tiles])
    pairs = (sz[:, None] * sz[None, :])[iu][keep[iu]].sum()
    return int(keep[iu].sum()), len(iu[0]), int(pairs)
tiles = [perm[i:i + 128] for i in range(0, n, 128)]
print("current: kept tiles, total, pairs", kept_pairs(tiles), flush=True)
# split at group transitions whose seeds are far apart (full-D seed distance > 2 eps)
Dfull = np.sqrt(((seeds[:, None, :] - seeds[None, :, :]) ** 2).sum(-1))
ks = key[perm]
tiles2 = []; cur_t = []
breaks = 0
for i, p in enumerate(perm):
    if cur_t and ks[i] != ks[i - 1]:
        a, b = order[ks[i - 1]], order[ks[i]]
        if Dfull[a, b] > 2 * eps:
            tiles2.append(np.array(cur_t)); cur_t = []; breaks += 1
    cur_t.append(p)
    if len(cur_t) == 128:
        tiles2.append(np.array(cur_t)); cur_t = []
if cur_t: tiles2.append(np.array(cur_t))
print("split at far transitions:", breaks, "breaks, tiles", len(tiles2), "vs", len(tiles), "kept", kept_pairs(tiles2), flush=True)
# every group on its own tiles
tiles3 = []; cur_t = []
for i, p in enumerate(perm):
    if cur_t and ks[i] != ks[i - 1]:
        tiles3.append(np.array(cur_t)); cur_t = []
    cur_t.append(p)
    if len(cur_t) == 128:
        tiles3.append(np.array(cur_t)); cur_t = []
if cur_t: tiles3.append(np.array(cur_t))
print("every group split: tiles", len(tiles3), "kept", kept_pairs(tiles3), flush=True)
