"""Seeded geometry and density generators for BASELINE.json configs[0..4].

All outputs are float32 arrays (the precision the CUDA path consumes); the oracle
promotes the same float32 values to fp64, so both sides see identical inputs.
"""
from __future__ import annotations

import numpy as np


def _f32(*arrs):
    return tuple(np.ascontiguousarray(a, dtype=np.float32) for a in arrs)


# ------------------------------------------------------------------ config 0
def sphere_points(n: int, seed: int = 0, radius: float = 1.0) -> np.ndarray:
    """n points uniform on the sphere (normalised Gaussian vectors)."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return np.ascontiguousarray(radius * v, dtype=np.float32)


def config0(n: int = 2048, seed: int = 0):
    """configs[0]: Kelvin single layer, N sources = targets uniform on the unit sphere,
    densities uniform in [-1, 1], K = 1.0, G = 0.5, self-interaction excluded."""
    pts = sphere_points(n, seed)
    rng = np.random.default_rng(seed + 1)
    f = rng.uniform(-1.0, 1.0, (n, 3))
    nrm = pts.astype(np.float64) / np.linalg.norm(pts.astype(np.float64), axis=1, keepdims=True)
    w = np.full(n, 4.0 * np.pi / n)
    pts, nrm, w, f = _f32(pts, nrm, w, f)
    return dict(src=pts, trg=pts, nrm=nrm, w=w, f=f, g=None, K=1.0, G=0.5)


# ------------------------------------------------------------------ triangle meshes
def cube_voxel_faces(nc: int, lo=(0.0, 0.0, 0.0), size=1.0):
    """surface of an axis-aligned cube split into nc x nc cells per face, each cell fanned
    into 4 triangles from its centre (Sec. 3: "Each side of the cell
    that belongs to a cube boundary is discretized onto 4 triangles", 24 N^2 in total).
    Returns (V0, V1, V2) vertex arrays with counter-clockwise order seen from outside."""
    tris = []
    h = size / nc
    lo = np.asarray(lo, np.float64)
    for axis in range(3):
        u, v = [a for a in range(3) if a != axis]
        for side in (0, 1):
            i, j = np.meshgrid(np.arange(nc), np.arange(nc), indexing="ij")
            i = i.reshape(-1).astype(np.float64)
            j = j.reshape(-1).astype(np.float64)
            corners = []
            for di, dj in ((0, 0), (1, 0), (1, 1), (0, 1)):
                p = np.zeros((i.size, 3))
                p[:, axis] = lo[axis] + side * size
                p[:, u] = lo[u] + (i + di) * h
                p[:, v] = lo[v] + (j + dj) * h
                corners.append(p)
            ctr = sum(corners) / 4.0
            # outward orientation: (u x v) = +axis for a cyclic (axis, u, v); flip as needed
            cyc = (u - axis) % 3 == 1
            flip = (side == 0) == cyc
            for k in range(4):
                a, b = corners[k], corners[(k + 1) % 4]
                tris.append((ctr, b, a) if flip else (ctr, a, b))
    V0 = np.concatenate([t[0] for t in tris])
    V1 = np.concatenate([t[1] for t in tris])
    V2 = np.concatenate([t[2] for t in tris])
    return V0, V1, V2


def panels(V0, V1, V2):
    """centroids, unit normals (right-hand rule) and areas of flat triangles."""
    c = (V0 + V1 + V2) / 3.0
    cr = np.cross(V1 - V0, V2 - V0)
    a2 = np.linalg.norm(cr, axis=1)
    return c, cr / a2[:, None], 0.5 * a2


def config1(nc: int = 32, seed: int = 1):
    """configs[1]: double-layer traction kernel on a triangulated unit cube surface,
    24,576 flat triangles (nc = 32 cells per edge, 4-triangle fan per cell = 24 nc^2,
    the paper's own cube discretisation; reading R7), collocation at
    centroids, outward normals, areas as weights, densities N(0,1), K = 1.67, G = 0.77."""
    V0, V1, V2 = cube_voxel_faces(nc)
    c, n, a = panels(V0, V1, V2)
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((c.shape[0], 3))
    c, n, a, g = _f32(c, n, a, g)
    return dict(src=c, trg=c, nrm=n, w=a, f=None, g=g, K=1.67, G=0.77)


def graded_beam_panels(h0: float, length=4.0, grade=4.0):
    """quad-split panels on the surface of the box [0,L]x[0,1]x[0,1], clamped end x = 0,
    panel size h(x) = h0 (1 + (grade-1) x / L): `grade` times finer at x = 0 than at x = L.
    Each slab [x_i, x_{i+1}] of a long face carries m_i = round(1/h_i) cells across; each
    rectangle is split into 2 triangles.  Returns centroids, outward normals, areas."""
    xs = [0.0]
    while xs[-1] < length:
        xs.append(xs[-1] + h0 * (1.0 + (grade - 1.0) * xs[-1] / length))
    xs = np.array(xs) * (length / xs[-1])
    C, N, A = [], [], []

    def rect_tris(p0, du, dv, nu_, nv_, normal):
        i, j = np.meshgrid(np.arange(nu_), np.arange(nv_), indexing="ij")
        i = i.reshape(-1, 1).astype(np.float64)
        j = j.reshape(-1, 1).astype(np.float64)
        a = p0 + i * du + j * dv
        b = a + du
        c = a + du + dv
        d = a + dv
        for t0, t1, t2 in ((a, b, c), (a, c, d)):
            C.append((t0 + t1 + t2) / 3.0)
            N.append(np.broadcast_to(normal, t0.shape))
            A.append(np.full(t0.shape[0], 0.5 * np.linalg.norm(np.cross(du, dv))))

    for s in range(len(xs) - 1):
        x0, x1 = xs[s], xs[s + 1]
        m = max(1, int(round(1.0 / (x1 - x0))))
        dx = np.array([x1 - x0, 0, 0])
        for (p0, dv, nrm) in (((x0, 0, 0), (0, 1.0 / m, 0), (0, 0, -1)),
                              ((x0, 0, 1), (0, 1.0 / m, 0), (0, 0, 1)),
                              ((x0, 0, 0), (0, 0, 1.0 / m), (0, -1, 0)),
                              ((x0, 1, 0), (0, 0, 1.0 / m), (0, 1, 0))):
            rect_tris(np.array(p0, float), dx, np.array(dv), 1, m, np.array(nrm, float))
    for xe, nrm, h in ((0.0, -1.0, h0), (length, 1.0, h0 * grade)):
        m = max(1, int(round(1.0 / h)))
        rect_tris(np.array([xe, 0, 0.0]), np.array([0, 1.0 / m, 0]), np.array([0, 0, 1.0 / m]), m, m,
                  np.array([nrm, 0, 0]))
    return np.concatenate(C), np.concatenate(N), np.concatenate(A)


def beam_h0_for(n_target: int) -> float:
    """panel size at the clamped end giving about n_target panels (total ~ 10.1 / h0^2)."""
    return float(np.sqrt(10.125 / n_target))


def smooth_density(points, seed: int, n_modes: int = 8, kmax: float = 2.0):
    """"solved-like" smooth density: sum of n_modes random low-frequency sinusoids per
    component (BASELINE.json configs[3])."""
    rng = np.random.default_rng(seed)
    p = np.asarray(points, np.float64)
    out = np.zeros((p.shape[0], 3))
    for c in range(3):
        for _ in range(n_modes):
            k = rng.uniform(-kmax, kmax, 3) * np.pi / 2
            ph = rng.uniform(0, 2 * np.pi)
            amp = rng.standard_normal()
            out[:, c] += amp * np.sin(p @ k + ph)
    return out


def config2(n: int = 200_000, seed: int = 2):
    """configs[2]: KIFMM matvec (single + double layer) on the 4x1x1 cantilever-beam
    surface, ~n centroid points graded 4x finer toward the clamped end, densities N(0,1),
    K = 1.67, G = 0.77 (max 64 points per leaf; p = 6 and p = 10 are run parameters)."""
    c, nrm, a = graded_beam_panels(beam_h0_for(n))
    rng = np.random.default_rng(seed)
    f = rng.standard_normal((c.shape[0], 3))
    g = rng.standard_normal((c.shape[0], 3))
    c, nrm, a, f, g = _f32(c, nrm, a, f, g)
    return dict(src=c, trg=c, nrm=nrm, w=a, f=f, g=g, K=1.67, G=0.77)


def interior_grid(nx=200, ny=50, nz=100, length=4.0, min_dist=1e-3):
    """regular nx x ny x nz cell-centre grid in [0,L]x[0,1]x[0,1] minus points within
    min_dist of the boundary (BASELINE.json configs[3])."""
    x = (np.arange(nx) + 0.5) * length / nx
    y = (np.arange(ny) + 0.5) / ny
    z = (np.arange(nz) + 0.5) / nz
    X, Y, Z = np.meshgrid(x, y, z, indexing="ij")
    p = np.stack([X, Y, Z], -1).reshape(-1, 3)
    d = np.minimum.reduce([p[:, 0], length - p[:, 0], p[:, 1], 1 - p[:, 1], p[:, 2], 1 - p[:, 2]])
    return p[d >= min_dist]


def config3(n_src: int = 500_000, grid=(200, 50, 100), seed: int = 3):
    """configs[3]: stress evaluation for the topological derivative: ~n_src beam surface
    sources with smooth densities (traction-like f and displacement-like g), interior
    targets on a regular grid, 6-component stress out, p = 8."""
    c, nrm, a = graded_beam_panels(beam_h0_for(n_src))
    f = smooth_density(c, seed)
    g = smooth_density(c, seed + 100)
    trg = interior_grid(*grid)
    c, nrm, a, f, g, trg = _f32(c, nrm, a, f, g, trg)
    return dict(src=c, trg=trg, nrm=nrm, w=a, f=f, g=g, K=1.67, G=0.77)


# ------------------------------------------------------------------ config 4 (GMRES)
def icosphere(level: int):
    """unit icosphere: icosahedron, each face split into 4 `level` times, vertices projected
    to the sphere.  Returns (V0, V1, V2) counter-clockwise seen from outside."""
    t = (1.0 + 5 ** 0.5) / 2.0
    verts = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
             (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
             (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5), (2, 4, 11),
             (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    V = np.array(verts, np.float64)
    V /= np.linalg.norm(V, axis=1, keepdims=True)
    F = np.array(faces)
    for _ in range(level):
        a, b, c = V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]
        ab, bc, ca = (a + b), (b + c), (c + a)
        ab /= np.linalg.norm(ab, axis=1, keepdims=True)
        bc /= np.linalg.norm(bc, axis=1, keepdims=True)
        ca /= np.linalg.norm(ca, axis=1, keepdims=True)
        nv = len(V)
        nf = len(F)
        V = np.concatenate([V, ab, bc, ca])
        iab, ibc, ica = nv + np.arange(nf), nv + nf + np.arange(nf), nv + 2 * nf + np.arange(nf)
        F = np.concatenate([np.stack([F[:, 0], iab, ica], 1), np.stack([F[:, 1], ibc, iab], 1),
                            np.stack([F[:, 2], ica, ibc], 1), np.stack([iab, ibc, ica], 1)])
    V0, V1, V2 = V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]
    # orient counter-clockwise seen from outside (outward normal)
    flip = np.einsum("ij,ij->i", np.cross(V1 - V0, V2 - V0), V0 + V1 + V2) < 0
    V1, V2 = np.where(flip[:, None], V2, V1), np.where(flip[:, None], V1, V2)
    return V0, V1, V2


def metamaterial_cell(nc=160, level=5, nvoids=64, rmin=0.05, rmax=0.1, gap=0.01, seed=4):
    """configs[4]: unit cube with `nvoids` seeded non-overlapping spherical voids of radius
    in [rmin, rmax], each an icosphere of `level`; the outer cube is meshed like configs[1]
    (nc cells per edge, 4-triangle fan).  Void surfaces are oriented with the normal out
    of the material (into the void).  Boundary conditions: Dirichlet u = 0 on the bottom
    face z = 0, Neumann traction (0, 0, -1) on the top face z = 1, traction free elsewhere.
    Returns dict(verts (n,3,3) float32, bc_type int32, bc_val float32 (n,3), K, G)."""
    rng = np.random.default_rng(seed)
    centers, radii = [], []
    tries = 0
    while len(centers) < nvoids:
        tries += 1
        if tries > 200000:
            raise RuntimeError("could not place the voids")
        r = rng.uniform(rmin, rmax)
        c = rng.uniform(r + gap, 1 - r - gap, 3)
        if all(np.linalg.norm(c - c2) > r + r2 + gap for c2, r2 in zip(centers, radii)):
            centers.append(c)
            radii.append(r)
    C0, C1, C2 = cube_voxel_faces(nc)
    S0, S1, S2 = icosphere(level)
    parts0, parts1, parts2 = [C0], [C1], [C2]
    for c, r in zip(centers, radii):
        # into the void: reverse the sphere's outward orientation
        parts0.append(c + r * S0)
        parts1.append(c + r * S2)
        parts2.append(c + r * S1)
    V0, V1, V2 = (np.concatenate(p) for p in (parts0, parts1, parts2))
    cen = (V0 + V1 + V2) / 3.0
    ncube = len(C0)
    bc = np.ones(len(V0), np.int32)
    val = np.zeros((len(V0), 3))
    bottom = np.zeros(len(V0), bool)
    bottom[:ncube] = cen[:ncube, 2] < 1e-9
    top = np.zeros(len(V0), bool)
    top[:ncube] = cen[:ncube, 2] > 1 - 1e-9
    bc[bottom] = 0
    val[top] = (0.0, 0.0, -1.0)
    verts = np.stack([V0, V1, V2], 1).astype(np.float32)
    return dict(verts=verts, bc_type=bc, bc_val=val.astype(np.float32), K=1.67, G=0.77,
                centers=np.array(centers), radii=np.array(radii))
