"""Seeded synthetic 2-D lidar worlds and scans -- the shared input generator.

This module is the ONLY thing the oracle and the CUDA path share: it holds no
arithmetic of the method (no phases, phasors, similarities or entropies), only
the world, sensor poses, ray casting and labelling that produce the labelled
point clouds (gamma, psi) of the paper's data format (sec. III-B-2).

The paper's own workloads (the BHM-simulator lidar set P:409-411, the Intel
Campus log P:507, the EviLOG data P:565) are not available; these synthetic
configurations stand in for them, following the paper's simulated-lidar style
(2-D beams, hits labelled occupied, free space sampled along beams) at
the scales of BASELINE.json configs C1..C5.  The recipe is SURVEY.md 8(d) and
is restated in DESIGN.md ("Input recipe").

Points are emitted per scan, per beam: the hit (label 1) then its free samples
(label 0).  A beam that reaches max range without a hit emits only free
samples drawn along the full range.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------- configs

CONFIGS = {
    # name: world, obstacles, sensor, method parameters, grid, window
    "C1": dict(W=10.0, n_obst=6, shapes="rect", poses="fixed", n_scans=1, beams=360, fov_deg=360.0,
               max_range=8.0, sigma=0.0, n_free=4, D=512, l=0.2, rows=100, cols=100, res=0.1,
               half=1, batch_scans=None, n_points=None),
    "C2": dict(W=40.0, n_obst=40, shapes="mix", poses="walk", n_scans=20, beams=1081, fov_deg=270.0,
               max_range=30.0, sigma=0.02, n_free=2, D=2048, l=0.25, rows=400, cols=400, res=0.1,
               half=2, batch_scans=None, n_points=None),
    "C3": dict(W=100.0, n_obst=300, shapes="mix", poses="iid", n_scans=1000, beams=1081, fov_deg=270.0,
               max_range=30.0, sigma=0.02, n_free=1, D=4096, l=0.3, rows=1000, cols=1000, res=0.1,
               half=2, batch_scans=None, n_points=None),
    "C4": dict(W=100.0, n_obst=300, shapes="mix", poses="iid", n_scans=5000, beams=1081, fov_deg=270.0,
               max_range=30.0, sigma=0.02, n_free=1, D=8192, l=0.3, rows=2000, cols=2000, res=0.05,
               half=2, batch_scans=100, n_points=None),
    "C5": dict(W=200.0, n_obst=2000, shapes="mix", poses="iid", n_scans=None, beams=1081, fov_deg=270.0,
               max_range=30.0, sigma=0.02, n_free=2, D=16384, l=0.3, rows=4000, cols=4000, res=0.05,
               half=3, batch_scans=None, n_points=10_000_000),
}


@dataclass
class World:
    W: float
    rects: np.ndarray = field(default_factory=lambda: np.zeros((0, 4)))    # xmin, ymin, xmax, ymax
    circles: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))  # cx, cy, r

    def inside_obstacle(self, x: float, y: float) -> bool:
        r = self.rects
        if len(r) and np.any((x >= r[:, 0]) & (x <= r[:, 2]) & (y >= r[:, 1]) & (y <= r[:, 3])):
            return True
        c = self.circles
        if len(c) and np.any((x - c[:, 0]) ** 2 + (y - c[:, 1]) ** 2 <= c[:, 2] ** 2):
            return True
        return False


def make_world(cfg: dict, rng: np.random.Generator, keep_clear=None) -> World:
    """Random axis-aligned rectangles (sides U(0.5, 3) m) and, for "mix", circles
    (radius U(0.25, 1.5) m) by a fair coin; centres uniform in the world.  An
    obstacle containing ``keep_clear`` (the fixed sensor / walk start) is re-drawn."""
    W = cfg["W"]
    rects, circles = [], []
    while len(rects) + len(circles) < cfg["n_obst"]:
        cx, cy = rng.uniform(0, W, size=2)
        is_rect = cfg["shapes"] == "rect" or rng.random() < 0.5
        if is_rect:
            sx, sy = rng.uniform(0.5, 3.0, size=2)
            o = (cx - sx / 2, cy - sy / 2, cx + sx / 2, cy + sy / 2)
            if keep_clear is not None and o[0] <= keep_clear[0] <= o[2] and o[1] <= keep_clear[1] <= o[3]:
                continue
            rects.append(o)
        else:
            r = rng.uniform(0.25, 1.5)
            if keep_clear is not None and (keep_clear[0] - cx) ** 2 + (keep_clear[1] - cy) ** 2 <= r * r:
                continue
            circles.append((cx, cy, r))
    return World(W=W, rects=np.array(rects, dtype=np.float64).reshape(-1, 4),
                 circles=np.array(circles, dtype=np.float64).reshape(-1, 3))


def make_poses(cfg: dict, world: World, rng: np.random.Generator, n_scans: int) -> np.ndarray:
    """Sensor poses (x, y, heading) [n_scans, 3]."""
    W = cfg["W"]
    if cfg["poses"] == "fixed":
        return np.array([[W / 2, W / 2, 0.0]] * n_scans)
    out = []
    if cfg["poses"] == "walk":
        x, y = W / 2, W / 2
        h = rng.uniform(-math.pi, math.pi)
        out.append((x, y, h))
        while len(out) < n_scans:
            h = rng.uniform(-math.pi, math.pi)
            nx, ny = x + 1.5 * math.cos(h), y + 1.5 * math.sin(h)
            if not (0.5 <= nx <= W - 0.5 and 0.5 <= ny <= W - 0.5) or world.inside_obstacle(nx, ny):
                continue
            x, y = nx, ny
            out.append((x, y, h))
        return np.array(out)
    while len(out) < n_scans:          # iid uniform in free space, uniform heading
        x, y = rng.uniform(0.5, W - 0.5, size=2)
        h = rng.uniform(-math.pi, math.pi)
        if world.inside_obstacle(x, y):
            continue
        out.append((x, y, h))
    return np.array(out)


def cast(world: World, ox: float, oy: float, ang: np.ndarray, max_range: float) -> np.ndarray:
    """Distance to the first wall/obstacle along each beam, inf if beyond max_range."""
    dx, dy = np.cos(ang), np.sin(ang)
    with np.errstate(divide="ignore", invalid="ignore"):
        # boundary walls of [0, W]^2
        tx = np.where(dx > 0, (world.W - ox) / dx, np.where(dx < 0, -ox / dx, np.inf))
        ty = np.where(dy > 0, (world.W - oy) / dy, np.where(dy < 0, -oy / dy, np.inf))
        t = np.minimum(tx, ty)
        reach = max_range + 3.0
        r = world.rects
        if len(r):
            near = (np.maximum(np.maximum(r[:, 0] - ox, ox - r[:, 2]), 0) ** 2
                    + np.maximum(np.maximum(r[:, 1] - oy, oy - r[:, 3]), 0) ** 2) <= reach ** 2
            r = r[near]
        if len(r):
            idx = 1.0 / dx[:, None]
            idy = 1.0 / dy[:, None]
            t1 = (r[None, :, 0] - ox) * idx
            t2 = (r[None, :, 2] - ox) * idx
            t3 = (r[None, :, 1] - oy) * idy
            t4 = (r[None, :, 3] - oy) * idy
            tmin = np.maximum(np.minimum(t1, t2), np.minimum(t3, t4))
            tmax = np.minimum(np.maximum(t1, t2), np.maximum(t3, t4))
            hit = (tmax >= tmin) & (tmin > 0)
            t = np.minimum(t, np.where(hit, tmin, np.inf).min(axis=1))
        c = world.circles
        if len(c):
            near = (c[:, 0] - ox) ** 2 + (c[:, 1] - oy) ** 2 <= (reach + c[:, 2]) ** 2
            c = c[near]
        if len(c):
            fx = ox - c[None, :, 0]
            fy = oy - c[None, :, 1]
            b = dx[:, None] * fx + dy[:, None] * fy
            cc = fx * fx + fy * fy - c[None, :, 2] ** 2
            disc = b * b - cc
            tc = -b - np.sqrt(np.where(disc >= 0, disc, 0))
            tc = np.where((disc >= 0) & (tc > 0), tc, np.inf)
            t = np.minimum(t, tc.min(axis=1))
    return np.where(t <= max_range, t, np.inf)


def scan_points(cfg: dict, world: World, pose, rng_noise, rng_free):
    """One scan -> (xy float64 [n, 2], labels uint8 [n]) in beam order: hit, then free samples."""
    ox, oy, h = pose
    nb = cfg["beams"]
    if cfg["fov_deg"] >= 360.0:
        ang = 2 * math.pi * np.arange(nb) / nb
    else:
        half = math.radians(cfg["fov_deg"]) / 2
        ang = h + np.linspace(-half, half, nb)
    t = cast(world, ox, oy, ang, cfg["max_range"])
    hit = np.isfinite(t)
    meas = t.copy()
    if cfg["sigma"] > 0:
        meas[hit] += rng_noise.normal(0.0, cfg["sigma"], size=int(hit.sum()))
    span = np.where(hit, meas, cfg["max_range"])
    nf = cfg["n_free"]
    s = rng_free.uniform(0.0, 1.0, size=(nb, nf)) * span[:, None]
    per = 1 + nf
    xs = np.empty((nb, per))
    ys = np.empty((nb, per))
    lab = np.zeros((nb, per), dtype=np.uint8)
    xs[:, 0] = ox + meas * np.cos(ang)
    ys[:, 0] = oy + meas * np.sin(ang)
    lab[:, 0] = 1
    xs[:, 1:] = ox + s * np.cos(ang)[:, None]
    ys[:, 1:] = oy + s * np.sin(ang)[:, None]
    keep = np.ones((nb, per), dtype=bool)
    keep[:, 0] = hit
    xy = np.stack([xs[keep], ys[keep]], axis=1)
    return xy, lab[keep]


class Scenario:
    """World + poses for one config; scans are ray-cast on demand (deterministic)."""

    def __init__(self, name: str, seed: int = 0):
        self.name = name
        self.cfg = dict(CONFIGS[name])
        self.seed = seed
        ss = np.random.SeedSequence(seed)
        s_obst, s_pose, self._s_noise, self._s_free = ss.spawn(4)
        W = self.cfg["W"]
        clear = (W / 2, W / 2) if self.cfg["poses"] in ("fixed", "walk") else None
        self.world = make_world(self.cfg, np.random.default_rng(s_obst), keep_clear=clear)
        n_scans = self.cfg["n_scans"] or int(math.ceil(self.cfg["n_points"] / (self.cfg["beams"] * 1.5))) + 64
        self.poses = make_poses(self.cfg, self.world, np.random.default_rng(s_pose), n_scans)

    def _scan(self, j: int):
        # per-scan sub-streams so any scan range can be generated independently
        rn = np.random.default_rng(np.random.SeedSequence(self._s_noise.entropy,
                                                          spawn_key=self._s_noise.spawn_key + (j,)))
        rf = np.random.default_rng(np.random.SeedSequence(self._s_free.entropy,
                                                          spawn_key=self._s_free.spawn_key + (j,)))
        return scan_points(self.cfg, self.world, self.poses[j], rn, rf)

    def scans(self, j0: int, j1: int):
        xs, ls = [], []
        for j in range(j0, j1):
            xy, lab = self._scan(j)
            xs.append(xy)
            ls.append(lab)
        xy = np.concatenate(xs).astype(np.float32) if xs else np.zeros((0, 2), np.float32)
        lab = np.concatenate(ls) if ls else np.zeros(0, np.uint8)
        return np.ascontiguousarray(xy), np.ascontiguousarray(lab)

    def batch(self, b: int):
        """Streaming batch b (C4): scans [b*batch, (b+1)*batch)."""
        bs = self.cfg["batch_scans"] or len(self.poses)
        return self.scans(b * bs, (b + 1) * bs)

    def all_points(self):
        """The whole point cloud of the config (C5: truncated to exactly n_points)."""
        if self.cfg["n_points"] is None:
            return self.scans(0, len(self.poses))
        target = self.cfg["n_points"]
        xs, ls, n, j = [], [], 0, 0
        while n < target:
            if j >= len(self.poses):
                raise RuntimeError("not enough poses for the point target")
            xy, lab = self._scan(j)
            xs.append(xy.astype(np.float32))
            ls.append(lab)
            n += len(lab)
            j += 1
        xy = np.concatenate(xs)[:target]
        lab = np.concatenate(ls)[:target]
        return np.ascontiguousarray(xy), np.ascontiguousarray(lab)

    # grid / method parameters -------------------------------------------------
    @property
    def bounds(self):
        W = self.cfg["W"]
        return (0.0, 0.0, W, W)

    @property
    def grid(self):
        c = self.cfg
        return dict(x0=0.0, y0=0.0, res=c["res"], rows=c["rows"], cols=c["cols"])

