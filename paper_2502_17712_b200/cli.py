"""Mirror of the per-frame slice of atlaspack.cli (cli.py:209-406).

`run_scene_pipeline(cfg, packer="fastatlas")` keeps the reference
signature and SceneResult fields; the frame itself is one FrameEngine run
(csrc/, CUDA graph).  SceneResult's reference-typed fields (chart_set dicts,
boxes, layout, chart_ndc / chart_px dicts, stretch) are materialised lazily
from the device arrays.  The box / layout / charts file formats, SVG and
the `compare` / `gen-boxes` commands are outside the per-frame path
 and are not part of this package.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .charts import Mesh, load_obj
from .frame import FrameEngine, FrameOutput, FrameSettings
from .geometry import CameraFrame, W_EPSILON
from .packing import ChartBox, PackFailure, pack

EXIT_OK = 0
EXIT_BAD_INPUT = 1
EXIT_PACK_FAILURE = 2
EXIT_NOTHING_VISIBLE = 3

PACKER_NAMES = ("fastatlas", "sequential", "superblock")


class InputError(Exception):
    """Malformed input file; message names the offending record."""


class NothingVisible(Exception):
    """The camera sees no triangle at all."""


def generate_boxes(count: int, omega: int, rng: np.random.Generator) -> list:
    """cli.py:126-139: seeded heavy-tailed box set (test/bench input generator)."""
    u = rng.random((count, 2))
    dims = np.clip((omega * u ** 3).astype(np.int64), 1, omega)
    min_tris = rng.choice(max(count * 8, 8), size=count, replace=False)
    return [ChartBox(target_w=int(dims[i, 0]), target_h=int(dims[i, 1]), chart_id=i, min_tri=int(min_tris[i]))
            for i in range(count)]


@dataclass
class SceneConfig:
    """cli.py:209-239."""

    mesh_path: Path
    fov_y_deg: float = 60.0
    aspect: float | None = None
    near: float = 0.1
    far: float = 1000.0
    position: tuple = (0.0, 0.0, 0.0)
    look_at: tuple = (0.0, 0.0, -1.0)
    up: tuple = (0.0, 1.0, 0.0)
    screen: tuple = (1920, 1080)
    omega: int = 2048
    n_scales: int = 64
    min_dim: int = 1
    padding: int = 0
    backface_cull: bool = True
    prescale: float = 1.0

    def camera(self) -> CameraFrame:
        aspect = self.aspect if self.aspect is not None else self.screen[0] / self.screen[1]
        return CameraFrame.from_params(fov_y=math.radians(self.fov_y_deg), aspect=aspect, near=self.near,
                                       far=self.far, position=self.position, look_at=self.look_at, up=self.up)

    def frame_settings(self, **overrides) -> FrameSettings:
        s = FrameSettings(screen=tuple(self.screen), omega=self.omega, n_scales=self.n_scales, min_dim=self.min_dim,
                          padding=self.padding, prescale=self.prescale, backface_cull=self.backface_cull)
        for k, v in overrides.items():
            setattr(s, k, v)
        return s


def parse_scene_config(path) -> SceneConfig:
    """cli.py:242-308: key-value scene file, unknown keys rejected."""
    path = Path(path)
    values: dict = {}
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            key, *rest = line.split()
            if not rest:
                raise InputError(f"{path}:{lineno}: key '{key}' has no value")
            if key in values:
                raise InputError(f"{path}:{lineno}: duplicate key '{key}'")
            values[key] = rest

    def take(key, n, conv):
        rest = values.pop(key)
        if len(rest) != n:
            raise InputError(f"{path}: key '{key}' expects {n} values")
        out = tuple(conv(v) for v in rest)
        return out[0] if n == 1 else out

    try:
        if "mesh" not in values:
            raise InputError(f"{path}: missing required key 'mesh'")
        cfg = SceneConfig(mesh_path=(path.parent / values.pop("mesh")[0]).resolve())
        spec = [("fov_y", "fov_y_deg", 1, float), ("aspect", "aspect", 1, float), ("near", "near", 1, float),
                ("far", "far", 1, float), ("position", "position", 3, float), ("look_at", "look_at", 3, float),
                ("up", "up", 3, float), ("screen", "screen", 2, int), ("omega", "omega", 1, int),
                ("scales", "n_scales", 1, int), ("min_dim", "min_dim", 1, int), ("padding", "padding", 1, int),
                ("prescale", "prescale", 1, float)]
        for key, attr, n, conv in spec:
            if key in values:
                setattr(cfg, attr, take(key, n, conv))
        if "backface_cull" in values:
            cfg.backface_cull = take("backface_cull", 1, str).lower() in ("1", "true", "yes", "on")
    except (ValueError, KeyError) as exc:
        raise InputError(f"{path}: {exc}") from None
    if values:
        raise InputError(f"{path}: unknown keys: {', '.join(sorted(values))}")
    if cfg.omega & (cfg.omega - 1) or cfg.omega < 1:
        raise InputError(f"{path}: omega must be a power of two")
    if cfg.screen[0] < 1 or cfg.screen[1] < 1:
        raise InputError(f"{path}: screen must be at least 1x1")
    if not cfg.near < cfg.far:
        raise InputError(f"{path}: near must be less than far")
    return cfg


def make_packer(name: str, n_scales: int, min_dim: int, padding: int, block_size: int | None = None):
    """cli.py:318-339: the FastAtlas packer plus the comparison packers
    (csrc/fa_baselines.cu), all on the GPU."""
    from .baselines import SuperblockConfig, sequential_scale_search, superblock_pack
    if name == "fastatlas":
        return lambda boxes, omega: pack(boxes, omega, n_scales=n_scales, min_dim=min_dim, padding=padding)
    if name == "sequential":
        return lambda boxes, omega: sequential_scale_search(boxes, omega, n_scales=n_scales, min_dim=min_dim,
                                                            padding=padding)
    if name == "superblock":
        def run(boxes, omega):
            cfg = SuperblockConfig(block_size=block_size or default_block_size(omega))
            layout = superblock_pack(boxes, omega, cfg)
            if layout is None:
                raise PackFailure("superblock allocation failed at the halving floor")
            return layout
        return run
    raise InputError(f"unknown packer '{name}' (choose from {', '.join(PACKER_NAMES)})")


def default_block_size(omega: int) -> int:
    """cli.py:314-315."""
    return max(16, min(omega, omega // 8))


class SceneResult:
    """cli.py:345-357, with the reference-typed fields materialised on access."""

    def __init__(self, config: SceneConfig, mesh: Mesh, out: FrameOutput, cam: CameraFrame):
        self.config = config
        self.mesh = mesh
        self.frame = out
        self.camera = cam
        self.screen_fragments = out.screen_fragments
        self.texels_allocated = out.texels_allocated
        self.n_visible = out.n_visible
        self._cache = {}

    def _get(self, key, fn):
        if key not in self._cache:
            self._cache[key] = fn()
        return self._cache[key]

    @property
    def chart_set(self):
        return self._get("cs", self.frame.chart_set)

    @property
    def boxes(self):
        return self._get("boxes", self.frame.boxes)

    @property
    def layout(self):
        return self._get("layout", self.frame.layout)

    @property
    def chart_ndc(self):
        return self._get("ndc", self.frame.chart_ndc)

    @property
    def chart_px(self):
        return self._get("px", self.frame.chart_px)

    @property
    def uv(self) -> np.ndarray:
        """(n_visible, 6) atlas UVs in ascending visible-triangle order (NaN rows: no UV)."""
        return self._get("uv", lambda: self.frame.uv.cpu().numpy())

    @property
    def visible(self) -> np.ndarray:
        return self._get("vis", lambda: self.frame.visible.cpu().numpy())

    @property
    def stretch(self):
        """cli.py:409-454: screen-vs-atlas stretch over fully projectable
        triangles, reduced on the GPU inside the UV kernel (csrc/fa_uv.cu)."""
        return self._get("stretch", self.frame.stretch)


def run_scene_pipeline(cfg: SceneConfig, packer: str = "fastatlas", mesh: Mesh | None = None,
                       engine: FrameEngine | None = None) -> SceneResult:
    """cli.py:360-406 on the GPU.  `mesh` skips OBJ parsing; `engine` reuses a
    resident FrameEngine (and its CUDA graph) across frames."""
    if mesh is None:
        mesh = engine.mesh if engine is not None else load_obj(cfg.mesh_path)
    cam = cfg.camera()
    if engine is None:
        engine = FrameEngine(mesh)
    # the packer runs on the GPU inside the frame (fa_frame_params.packer):
    # fastatlas in the frame's CUDA graph, sequential / superblock
    # (baselines.py) after one synchronisation on the box count.  As in the
    # reference, an unknown name fails only after the NothingVisible check.
    try:
        out = engine.run(cam.view_proj, cfg.frame_settings(packer=packer))
    except ValueError:
        if packer not in PACKER_NAMES:
            raise InputError(f"unknown packer '{packer}' (choose from {', '.join(PACKER_NAMES)})") from None
        raise
    return SceneResult(cfg, mesh, out, cam)


__all__ = ["EXIT_OK", "EXIT_BAD_INPUT", "EXIT_PACK_FAILURE", "EXIT_NOTHING_VISIBLE", "InputError", "NothingVisible",
           "SceneConfig", "SceneResult", "generate_boxes", "make_packer", "parse_scene_config",
           "run_scene_pipeline", "W_EPSILON", "PackFailure"]
