"""Synthetic inputs for the BASELINE.json configurations.

These are the data formats on either side of the solve path: partition
labels (one int per active node, consumed by the reference's
load_partition, proj/include/cpdd/partition.hpp:519-552) and right-hand
sides (one value per active node, consumed by the `rhs = file:PATH` branch of
resolve_rhs, proj/include/cpdd/pipeline.hpp:103-117).  All randomness comes
from splitmix64 with explicit mappings, never from library distributions, so
every input is reproducible bit for bit on any host.
"""
from __future__ import annotations

import math

import numpy as np

_MASK = (1 << 64) - 1


class SplitMix64:
    """splitmix64 (Steele, Lea, Flood 2014) with explicit float mappings."""

    def __init__(self, seed: int):
        self.s = seed & _MASK

    def next_u64(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & _MASK
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def uniform(self) -> float:
        """Uniform on [0, 1): top 53 bits."""
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)

    def randint(self, lo: int, hi: int) -> int:
        """Integer in [lo, hi] by rejection-free multiply-shift (hi-lo+1 << 2^32)."""
        span = hi - lo + 1
        return lo + ((self.next_u64() >> 32) * span >> 32)

    def normal(self) -> float:
        """Standard normal by Box-Muller (cosine branch), two uniforms per draw."""
        u1 = self.uniform()
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(1.0 - u1)) * math.cos(2.0 * math.pi * u2)


def uniform_vector(n: int, seed: int) -> np.ndarray:
    """x ~ U(-1, 1), seeded (operator/preconditioner parity inputs)."""
    g = SplitMix64(seed)
    return np.array([2.0 * g.uniform() - 1.0 for _ in range(n)])


# ----------------------------------------------------------------- partitions

def sector_partition(cp: np.ndarray, n_parts: int) -> np.ndarray:
    """Angular sectors of the closest points (BASELINE config 1):
    part = floor(n * theta / 2pi), theta = atan2(y, x) in [0, 2pi)."""
    th = np.arctan2(cp[:, 1], cp[:, 0])
    th = np.where(th < 0, th + 2 * np.pi, th)
    part = np.floor(n_parts * th / (2 * np.pi)).astype(np.int64)
    return np.clip(part, 0, n_parts - 1).astype(np.int32)


def rcb_partition(cp: np.ndarray, n_parts: int) -> np.ndarray:
    """Recursive coordinate bisection of the active closest points
    (BASELINE configs 2-5): split along the axis of longest extent, at the
    rank proportional to the part counts of the two halves, ordering points
    stably by (coordinate, active ordinal)."""
    n = cp.shape[0]
    part = np.zeros(n, np.int32)
    stack = [(np.arange(n, dtype=np.int64), n_parts, 0)]
    while stack:
        idx, k, base = stack.pop()
        if k == 1 or idx.size == 0:
            part[idx] = base
            continue
        pts = cp[idx]
        ext = pts.max(axis=0) - pts.min(axis=0)
        axis = int(np.argmax(ext))
        order = np.lexsort((idx, pts[:, axis]))
        k1 = k // 2
        cut = (idx.size * k1 + k // 2) // k
        left, right = idx[order[:cut]], idx[order[cut:]]
        stack.append((right, k - k1, base + k1))
        stack.append((left, k1, base))
    return part


# ----------------------------------------------------------- right-hand sides

def rhs_circle(cp: np.ndarray) -> np.ndarray:
    """Config 1: f = 2 sin(theta) + 145 sin(12 theta) for u = sin(theta) + sin(12 theta), c = 1."""
    th = np.arctan2(cp[:, 1], cp[:, 0])
    return 2.0 * np.sin(th) + 145.0 * np.sin(12.0 * th)


def exact_circle(cp: np.ndarray) -> np.ndarray:
    th = np.arctan2(cp[:, 1], cp[:, 0])
    return np.sin(th) + np.sin(12.0 * th)


def exact_sphere(cp: np.ndarray) -> np.ndarray:
    """Configs 2-3: u = sin^3(theta) cos(3 phi) = x^3 - 3 x y^2 on the unit sphere
    (theta polar, phi azimuth); a degree-3 harmonic, so (1 - Lap_S) u = 13 u."""
    r = np.linalg.norm(cp, axis=1)
    x, y = cp[:, 0] / r, cp[:, 1] / r
    return x ** 3 - 3.0 * x * y * y


def rhs_sphere(cp: np.ndarray) -> np.ndarray:
    return 13.0 * exact_sphere(cp)


def trig_modes(seed: int, n_modes: int = 16):
    """k_m integer in [-4, 4]^3, phi_m uniform on [0, 2 pi) (configs 4-5)."""
    g = SplitMix64(seed)
    ks = np.array([[g.randint(-4, 4) for _ in range(3)] for _ in range(n_modes)], np.float64)
    ph = np.array([2.0 * np.pi * g.uniform() for _ in range(n_modes)])
    return ks, ph


def rhs_trig(cp: np.ndarray, seed: int, n_modes: int = 16) -> np.ndarray:
    ks, ph = trig_modes(seed, n_modes)
    f = np.zeros(cp.shape[0])
    for k, p in zip(ks, ph):
        f += np.sin(cp @ k + p)
    return f


def write_vector(path: str, v: np.ndarray) -> None:
    """One value per line, %.17g (round-trips exactly through operator>>)."""
    with open(path, "w") as fh:
        fh.write("".join(f"{x:.17g}\n" for x in v))


def write_partition(path: str, part: np.ndarray) -> None:
    with open(path, "w") as fh:
        fh.write("".join(f"{int(p)}\n" for p in part))


# ------------------------------------------------------------ triangle mesh

def icosphere(subdivisions: int):
    """Unit icosphere: the icosahedron with each triangle split into four,
    midpoints projected to the sphere, `subdivisions` times (6 -> 40962
    vertices, 81920 triangles; BASELINE config 5)."""
    t = (1.0 + math.sqrt(5.0)) / 2.0
    verts = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
             (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    verts = [tuple(c / math.sqrt(sum(q * q for q in v)) for c in v) for v in verts]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
             (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5), (2, 4, 11),
             (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdivisions):
        cache = {}

        def mid(a, b):
            key = (a, b) if a < b else (b, a)
            if key not in cache:
                va, vb = verts[a], verts[b]
                m = [(va[i] + vb[i]) * 0.5 for i in range(3)]
                r = math.sqrt(sum(q * q for q in m))
                verts.append(tuple(q / r for q in m))
                cache[key] = len(verts) - 1
            return cache[key]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    return np.array(verts, np.float64), np.array(faces, np.int64)


def real_sph_harm(l: int, m: int, theta: np.ndarray, phi: np.ndarray) -> np.ndarray:
    """Orthonormal real spherical harmonic Y_lm (theta polar, phi azimuth)."""
    from scipy.special import lpmv
    am = abs(m)
    norm = math.sqrt((2 * l + 1) / (4 * math.pi) * math.factorial(l - am) / math.factorial(l + am))
    p = lpmv(am, l, np.cos(theta))
    if m == 0:
        return norm * p
    fac = math.sqrt(2.0) * norm * p
    return fac * (np.cos(am * phi) if m > 0 else np.sin(am * phi))


def displaced_icosphere(subdivisions: int = 6, seed: int = 5, amplitude: float = 0.1, lmax: int = 4):
    """BASELINE config 5 surface: icosphere vertices displaced radially to
    r = 1 + amplitude * sum_{l<=lmax} a_lm Y_lm, a_lm ~ N(0,1)/(l+1) (seeded)."""
    v, f = icosphere(subdivisions)
    theta = np.arccos(np.clip(v[:, 2], -1.0, 1.0))
    phi = np.arctan2(v[:, 1], v[:, 0])
    g = SplitMix64(seed)
    r = np.ones(v.shape[0])
    for l in range(lmax + 1):
        for m in range(-l, l + 1):
            r += amplitude * (g.normal() / (l + 1)) * real_sph_harm(l, m, theta, phi)
    return v * r[:, None], f


def write_obj(path: str, verts: np.ndarray, faces: np.ndarray) -> None:
    """Wavefront OBJ (1-based faces), %.17g vertices (exact round trip)."""
    with open(path, "w") as fh:
        fh.write("".join(f"v {x:.17g} {y:.17g} {z:.17g}\n" for x, y, z in verts))
        fh.write("".join(f"f {a + 1} {b + 1} {c + 1}\n" for a, b, c in faces))
