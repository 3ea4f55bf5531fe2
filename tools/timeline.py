"""Region timeline from a region_crit dump (JV_CRIT_DUMP): start matrix,
cadence by wave index, lag behind the upstream regions.
python tools/timeline.py FILE.npz [grid_side]"""
import sys

import numpy as np

np.set_printoptions(linewidth=250, precision=1, suppress=True)
z = np.load(sys.argv[1])
g = z['g'].astype(np.int64)
rw = z['rw']
wl = z['wl']
en = (g[:, 7] - g[:, 7].min()) / 1e3
nreg = len(rw) - 1
side = int(sys.argv[2]) if len(sys.argv) > 2 else int(round(nreg ** 0.5))
first = np.array([en[rw[r]] for r in range(nreg)])
last = np.array([en[rw[r + 1] - 1] for r in range(nreg)])
print('span', en.max())
if side * side == nreg:
    print('first-wave end times:')
    print(first.reshape(side, side))
prof = []
for r in range(nreg):
    d = np.diff(en[rw[r]:rw[r + 1]])
    prof.append([d[i:i + 10].mean() for i in range(0, len(d) - 9, 10)][:14])
m = min(len(p) for p in prof)
prof = np.array([p[:m] for p in prof])
np.set_printoptions(linewidth=250, precision=2, suppress=True)
print('mean wave time by wave-index decile (us), all regions:', prof.mean(0))
print('region 0:', prof[0])


def E(r):
    return en[rw[r]:rw[r + 1]]


def L(r):
    return wl[rw[r]:rw[r + 1]]


def at(rr, l):
    i = np.searchsorted(L(rr), l)
    return E(rr)[i] if i < len(L(rr)) and L(rr)[i] == l else np.nan


if side * side == nreg:
    lags = []
    for r in range(nreg):
        a, b = divmod(r, side)
        ups = ([r - side] if a else []) + ([r - 1] if b else [])
        if not ups:
            continue
        lg = []
        for w in range(0, len(L(r)), 5):
            t = np.nanmax([at(u, L(r)[w] - 1) for u in ups])
            if np.isfinite(t):
                lg.append(E(r)[w] - t)
        lags.append((np.median(lg), lg[0]))
    lags = np.array(lags)
    print('lag behind upstream (same level - 1): median over regions of median %.2f us, at first wave %.2f us' % (
        np.median(lags[:, 0]), np.median(lags[:, 1])))
