"""Seeded source selection for the BASELINE configs (shared input definition:
the same draws as the generator streams, see csrc/graph.cu)."""
import numpy as np

M64 = (1 << 64) - 1


def _mix64(z):
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M64
    z ^= z >> 31
    return z


def _stream(seed, stream):
    return _mix64(seed ^ _mix64((stream + 0x632BE59BD9B4E019) & M64))


def _draw(s, i):
    return _mix64((s + (i + 1) * 0x9E3779B97F4A7C15) & M64)


def pick_sources(deg, count, seed, stream=7):
    """`count` seeded sources among vertices with deg > 0, distinct while possible
    (BASELINE.json configs: "drawn from the seed among non-isolated vertices")."""
    deg = np.asarray(deg)
    n = len(deg)
    s = _stream(int(seed), stream)
    ok = int(np.count_nonzero(deg))
    out, seen = [], set()
    i = 0
    while len(out) < count and ok > 0:
        c = (_draw(s, i) * n) >> 64
        i += 1
        if deg[c] > 0 and (c not in seen or len(seen) >= ok):
            out.append(int(c))
            seen.add(int(c))
    return np.array(out, np.int64)
