"""The five BASELINE.json configurations as seeded synthetic inputs.

Mesh seed for config c, level l (1 = coarsest) is ``1000*c + l``; isolated
kernel input vectors are N(0,1) from ``default_rng(0)``.  ``scale`` divides the
cells per axis (rounded, >= 1) to produce smaller meshes of the same shape for
parity tests; scale=1 is the full configuration.
"""

from __future__ import annotations

from dataclasses import dataclass

from .mesh import jittered_box_mesh, sine_warp


@dataclass(frozen=True)
class ProblemConfig:
    name: str
    dim: int
    degree: int
    problem: str  # "poisson" | "elasticity"
    levels: tuple  # cells per axis per level, coarsest first
    extent: tuple
    amplitude: float
    warp: bool = False
    dirichlet_ids: object = "all"
    lame: tuple = None
    body_force: tuple = None
    chebyshev_degree: int = 4
    index: int = 0

    def level_grid(self, l, scale=1):
        g = self.levels[l]
        if scale == 1:
            return tuple(g)
        return tuple(max(1, int(round(n / scale))) for n in g)

    def make_meshes(self, scale=1, validate=True):
        out = []
        for l in range(len(self.levels)):
            out.append(
                jittered_box_mesh(
                    self.level_grid(l, scale),
                    self.extent,
                    self.amplitude,
                    seed=1000 * self.index + (l + 1),
                    warp=sine_warp if self.warp else None,
                    validate=validate,
                )
            )
        return out


UNIT2 = ((0.0, 1.0), (0.0, 1.0))
UNIT3 = ((0.0, 1.0), (0.0, 1.0), (0.0, 1.0))

CONFIGS = {
    "C1": ProblemConfig("C1", 2, 1, "poisson", ((17, 17), (45, 45), (128, 128)), UNIT2, 0.25,
                        index=1),
    "C2": ProblemConfig("C2", 2, 2, "poisson", ((64, 64), (181, 181), (512, 512)), UNIT2, 0.2,
                        index=2),
    "C3": ProblemConfig("C3", 3, 2, "poisson", ((17, 17, 17), (47, 47, 47), (128, 128, 128)),
                        UNIT3, 0.2, index=3),
    "C4": ProblemConfig("C4", 3, 4, "poisson", ((8, 8, 8), (23, 23, 23), (64, 64, 64)), UNIT3,
                        0.15, warp=True, index=4),
    "C5": ProblemConfig("C5", 3, 2, "elasticity", ((33, 4, 4), (93, 12, 12), (256, 32, 32)),
                        ((0.0, 8.0), (0.0, 1.0), (0.0, 1.0)), 0.2, dirichlet_ids=[0],
                        lame=(1.0, 1.0), body_force=(0.0, 0.0, -1.0), chebyshev_degree=5,
                        index=5),
}


def get_config(name):
    try:
        return CONFIGS[name.upper()]
    except KeyError:
        raise ValueError(f"unknown config {name!r}; choose from {sorted(CONFIGS)}") from None
