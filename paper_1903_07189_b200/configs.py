"""The five BASELINE.json configurations, with every generator parameter pinned
(DESIGN.md §6).  Seeded synthetic inputs stand in for the paper's images; no
dataset is named by BASELINE.json for this path."""
from __future__ import annotations

from dataclasses import dataclass

SEED_BASE = 0x1903_07189


@dataclass(frozen=True)
class WmcConfig:
    name: str
    w: int
    h: int
    planes: int          # channel planes (cfg3) or batch images (cfg5)
    iters: int           # 0 -> single WMC map evaluation (cfg1)
    n_rects: int
    n_discs: int
    sigma: float
    u8: bool = False
    dt: float = 1.0      # SPEC.md:251 default for half_laplace; BASELINE gives none
    sharding: str = "none"   # "rows" (cfg4) | "images" (cfg5) | "none"

    @property
    def pixels(self) -> int:
        return self.w * self.h * self.planes

    @property
    def updates(self) -> int:
        """pixel-updates per run (the metric's unit of work)."""
        return self.pixels * max(1, self.iters)

    def seed(self, plane: int) -> int:
        idx = int(self.name[3:].split("_")[0])
        return SEED_BASE + 1000 * idx + plane


CONFIGS = {
    "cfg1": WmcConfig("cfg1", 512, 512, 1, 0, 20, 20, 0.05),
    "cfg2": WmcConfig("cfg2", 1024, 1024, 1, 100, 20, 20, 0.10),
    "cfg3": WmcConfig("cfg3", 3840, 2160, 3, 50, 20, 20, 0.08),
    "cfg4": WmcConfig("cfg4", 16384, 16384, 1, 200, 2000, 2000, 0.10, sharding="rows"),
    "cfg5": WmcConfig("cfg5", 1920, 1080, 256, 20, 20, 20, 0.10, u8=True, sharding="images"),
}

# Not a BASELINE config: the map's HBM-roofline measurement on a large image
# (cfg1 is L2-resident and launch-bound, so the stencil's HBM
# claim comes from a supplemental 16384^2 single evaluation, cfg1's generator).
SUPPLEMENTAL = {
    "cfg1_16k": WmcConfig("cfg1_16k", 16384, 16384, 1, 0, 2000, 2000, 0.05),
}

