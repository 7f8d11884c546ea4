"""Seeded synthetic phantoms standing in for the paper's clinical MRI.

The paper's datasets are not available, so the five
BASELINE.json configurations are driven by these generators, built to the
shapes, sizes and value distributions SURVEY.md section 8(d) records.  A
phantom is defined on the full-resolution volume (``T = K + (K-1)(f-1)``
planes); the known slices are planes ``z = i*f`` and the withheld planes are
ground truth.  Only the requested planes are rasterised, so the benchmark can
build its K known slices without materialising the full volume.

Per-plane noise is drawn from ``default_rng([seed, z])``, so any subset of
planes is bit-identical to the same planes of the full volume.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from scipy.ndimage import gaussian_filter


@dataclass(frozen=True)
class PhantomConfig:
    name: str
    height: int
    width: int
    n_known: int
    factor: int
    n_subparts: int
    family: str                  # "head" | "spine" | "brain"
    seed: int
    blur: float
    rician: float
    quantise: str                # "u8" | "u12" | "f32"
    accum: str                   # kernel accumulation the config is quoted in
    n_shapes: int = 0            # ellipsoids (head) / lesions (brain)
    extra: dict = field(default_factory=dict, compare=False, hash=False)

    @property
    def depth(self) -> int:
        return self.n_known + (self.n_known - 1) * (self.factor - 1)

    @property
    def known_z(self) -> np.ndarray:
        return np.arange(self.n_known) * self.factor

    @property
    def interpolated_voxels(self) -> int:
        return ((self.n_known - 1) * (self.factor - 1) * self.height
                * self.width)


CONFIGS = {
    "C1": PhantomConfig("C1-head", 128, 128, 16, 2, 4, "head", 1, 1.0, 4.0,
                        "u8", "fp64", n_shapes=8),
    "C2": PhantomConfig("C2-spine", 256, 256, 32, 4, 8, "spine", 2, 1.2, 5.0,
                        "u8", "fp64"),
    "C3": PhantomConfig("C3-brain", 512, 512, 64, 4, 16, "brain", 3, 1.0,
                        0.02, "f32", "fp32", n_shapes=20),
    "C4": PhantomConfig("C4-hdr-spine", 512, 512, 256, 8, 32, "spine", 4, 1.2,
                        40.0, "u12", "fp64"),
    "C5": PhantomConfig("C5-large-brain", 1024, 1024, 512, 4, 64, "brain", 5,
                        1.0, 0.02, "f32", "fp32", n_shapes=100),
}


def small_config(family: str, height: int, width: int, n_known: int,
                 factor: int, n_subparts: int = 1, seed: int = 11,
                 quantise: str | None = None) -> PhantomConfig:
    """A reduced config of one family for parity tests."""
    q = quantise or {"head": "u8", "spine": "u8", "brain": "f32"}[family]
    rician = {"u8": 4.0, "u12": 40.0, "f32": 0.02}[q]
    return PhantomConfig(f"{family}-{height}x{width}x{n_known}-f{factor}",
                         height, width, n_known, factor, n_subparts, family,
                         seed, 1.0, rician, q, "fp64",
                         n_shapes=8 if family != "brain" else 6)


# --------------------------------------------------------------------------
# shape parameters (drawn once per config from default_rng(seed))
# --------------------------------------------------------------------------

def _shapes(cfg: PhantomConfig):
    rng = np.random.default_rng(cfg.seed)
    T, H, W = cfg.depth, cfg.height, cfg.width
    if cfg.family == "head":
        out = []
        for _ in range(cfg.n_shapes):
            c = rng.uniform([0, 0, 0], [W, H, T])
            ax = rng.uniform(10, 40, size=3)
            out.append((c, ax, rng.uniform(40, 230)))
        return out
    if cfg.family == "spine":
        n_vert = 12
        pitch = H / (2 * n_vert + 1)
        verts, discs = [], []
        for i in range(n_vert):
            yc = pitch * (2 * i + 1.5)
            verts.append((yc, rng.normal(200, 15)))
            if i < n_vert - 1:
                discs.append((yc + pitch, rng.normal(90, 10)))
        return {"pitch": pitch, "verts": verts, "discs": discs}
    # brain: lesions inside the white/grey matter
    lesions = []
    for _ in range(cfg.n_shapes):
        u = rng.uniform(-0.6, 0.6, size=3)
        c = np.array([W / 2 + u[0] * 0.40 * W, H / 2 + u[1] * 0.40 * H,
                      T / 2 + u[2] * 0.40 * T])
        lesions.append((c, rng.uniform(3, 10), rng.uniform(0.3, 1.0)))
    return lesions


def _clean_plane(cfg: PhantomConfig, shapes, z: float) -> np.ndarray:
    H, W, T = cfg.height, cfg.width, cfg.depth
    y, x = np.mgrid[0:H, 0:W].astype(np.float32)
    img = np.zeros((H, W), np.float32)
    if cfg.family == "head":
        for (c, ax, val) in shapes:
            dzn = (z - c[2]) / ax[2]
            if abs(dzn) >= 1.0:
                continue
            r = ((x - c[0]) / ax[0]) ** 2 + ((y - c[1]) / ax[1]) ** 2 + dzn ** 2
            img[r <= 1.0] = val
        return img
    if cfg.family == "spine":
        img[:] = 20.0
        pitch = shapes["pitch"]
        xc, zc = W * 0.5, T * 0.5
        zs = max(T * 0.45, 1.0)
        for (yc, val) in shapes["verts"]:            # rounded boxes
            u = np.abs((x - xc) / (0.20 * W))
            v = np.abs((y - yc) / (0.42 * pitch))
            w = abs((z - zc) / zs)
            img[u ** 4 + v ** 4 + w ** 4 <= 1.0] = val
        for (yc, val) in shapes["discs"]:            # elliptical discs
            u = (x - xc) / (0.19 * W)
            v = (y - yc) / (0.40 * pitch)
            w = (z - zc) / (0.9 * zs)
            img[u * u + v * v + w * w <= 1.0] = val
        cu = (x - (xc + 0.30 * W)) / (0.06 * W)       # cord along image y
        cw = (z - zc) / (0.5 * zs)
        img[cu * cu + cw * cw <= 1.0] = 140.0
        return img
    # brain: nested ellipsoid shells + lesions
    xc, yc, zc = W / 2, H / 2, T / 2
    for scale, val in ((0.46, 0.9), (0.42, 0.55), (0.34, 0.75)):
        r = (((x - xc) / (scale * W)) ** 2 + ((y - yc) / (scale * 1.12 * H))
             ** 2 + ((z - zc) / (scale * T)) ** 2)
        img[r <= 1.0] = val
    for dx in (-0.07, 0.07):                          # ventricles (CSF)
        r = (((x - xc - dx * W) / (0.05 * W)) ** 2 + ((y - yc) / (0.14 * H))
             ** 2 + ((z - zc) / (0.20 * T)) ** 2)
        img[r <= 1.0] = 0.2
    for (c, rad, val) in shapes:
        dzc = z - c[2]
        if abs(dzc) >= rad:
            continue
        r = (x - c[0]) ** 2 + (y - c[1]) ** 2 + dzc ** 2
        img[r <= rad * rad] = val
    return img


def phantom_planes(cfg: PhantomConfig, zs) -> np.ndarray:
    """Noisy, quantised planes ``zs`` of the phantom, float32 [len(zs),H,W]."""
    shapes = _shapes(cfg)
    out = np.empty((len(zs), cfg.height, cfg.width), np.float32)
    for i, z in enumerate(zs):
        img = _clean_plane(cfg, shapes, float(z))
        if cfg.quantise == "u12":
            img = img * np.float32(4095.0 / 255.0)
        img = gaussian_filter(img, cfg.blur, mode="nearest")
        rng = np.random.default_rng([cfg.seed, int(z)])
        n1 = rng.normal(0.0, cfg.rician, img.shape).astype(np.float32)
        n2 = rng.normal(0.0, cfg.rician, img.shape).astype(np.float32)
        img = np.sqrt((img + n1) ** 2 + n2 ** 2)
        if cfg.quantise == "u8":
            img = np.clip(np.rint(img), 0, 255)
        elif cfg.quantise == "u12":
            img = np.clip(np.rint(img), 0, 4095)
        else:
            img = np.clip(img, 0.0, 1.0)
        out[i] = img
    return out


def known_slices(cfg: PhantomConfig) -> np.ndarray:
    """The K known slices (planes z = i*f), float32 [K, H, W]."""
    return phantom_planes(cfg, cfg.known_z)


def ground_truth(cfg: PhantomConfig) -> np.ndarray:
    """The full-resolution volume, float32 [T, H, W] (small configs only)."""
    return phantom_planes(cfg, np.arange(cfg.depth))
