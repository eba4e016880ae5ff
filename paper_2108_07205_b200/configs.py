"""Synthetic stand-ins for the BASELINE.json configurations.

The paper's geometries (spline channel, Fallopian tube, star lattice) are not
available; the analytic curves named by BASELINE.json replace them.  All
random quantities come from numpy's default_rng(seed) on the host and are
handed identically to the device path and to the CPU oracle.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class RefinedWallConfig:
    name: str
    kind: str                 # "ellipse" | "star"
    n_panels: int
    q: int = 16
    a: float = 1.0            # ellipse semi-axes / star scale
    b: float = 1.0
    prongs: int = 5
    amplitude: float = 0.3
    eps: float = 1e-10
    leaf: int = 64
    n_refine: int = 4         # panels refined
    m: int = 8                # split factor (2^levels)
    refine_point: tuple | None = None
    nrhs: int = 1
    sources_per_rhs: int = 5
    seed: int = 0
    targets: int = 100

    # ------------------------------------------------------------ geometry
    def curve_eval(self, t):
        t = np.asarray(t, dtype=np.float64)
        if self.kind == "ellipse":
            return np.stack([self.a * np.cos(t), self.a * (self.b / self.a) * np.sin(t)], -1)
        r = 1.0 + self.amplitude * np.cos(self.prongs * t)
        return np.stack([self.a * r * np.cos(t), self.a * r * np.sin(t)], -1)

    def refine_target(self):
        if self.refine_point is not None:
            return np.asarray(self.refine_point, dtype=np.float64)
        rng = np.random.default_rng(self.seed + 1)
        return self.curve_eval(rng.uniform(0.0, 2 * np.pi))

    def refine_panels(self, nodes):
        """The n_refine panels with the smallest min-node distance to the target."""
        p = self.refine_target()
        d = np.hypot(nodes["x"] - p[0], nodes["y"] - p[1])
        pmin = np.full(self.n_panels, np.inf)
        np.minimum.at(pmin, nodes["panel_of"], d)
        return np.sort(np.argsort(pmin, kind="stable")[: self.n_refine])

    # ------------------------------------------------------------ data
    def sources(self):
        """Per RHS: Stokeslets (x, y, fx, fy) outside the domain, N(0,1) forces."""
        rng = np.random.default_rng(self.seed)
        out = []
        for j in range(self.nrhs):
            if self.name == "cfg1":
                ang = 2 * np.pi * np.arange(self.sources_per_rhs) / self.sources_per_rhs
                rad = np.full(self.sources_per_rhs, 4.0)
            else:
                ang = rng.uniform(0, 2 * np.pi, self.sources_per_rhs)
                rad = rng.uniform(1.5, 3.0, self.sources_per_rhs) * self.a
            f = rng.standard_normal((self.sources_per_rhs, 2))
            out.append(np.column_stack([rad * np.cos(ang), rad * np.sin(ang), f]))
        return out

    def interior_targets(self):
        """Seed-drawn interior points well away from the wall (inside the
        curve scaled by 0.7 about the origin)."""
        rng = np.random.default_rng(self.seed + 2)
        t = rng.uniform(0, 2 * np.pi, self.targets)
        s = 0.7 * np.sqrt(rng.uniform(0, 1, self.targets))
        return self.curve_eval(t) * s[:, None]


CONFIGS = {
    # BASELINE.json configs[0]: ellipse (2,1), 128x16 nodes, 4 panels near
    # (1.99, 0) split 3 dyadic levels (m = 8), 5 Stokeslets at radius 4.
    "cfg1": RefinedWallConfig("cfg1", "ellipse", 128, a=2.0, b=1.0, n_refine=4, m=8,
                              refine_point=(1.99, 0.0), nrhs=1, sources_per_rhs=5),
    # configs[1]: star 1 + 0.3 cos 5t, 1024x16 nodes, 16 panels near a seed
    # point split 4 levels (m = 16), 64 RHS of 8 exterior Stokeslets.
    "cfg2": RefinedWallConfig("cfg2", "star", 1024, a=1.0, n_refine=16, m=16, nrhs=64,
                              sources_per_rhs=8),
    # configs[2]: star, 4096x16 nodes, HBS inverse apply microbenchmark.
    "cfg3": RefinedWallConfig("cfg3", "star", 4096, a=1.0, n_refine=0, m=1, nrhs=1),
}
