"""Python host mirror of the reference `gsct` operator API, over the C ABI of
libgsct_b200.so (include/gsct_cuda.h) via ctypes.

Names, argument meaning and error behaviour follow the reference C++ library
(/root/reference/proj/include/gsct/): `rasterize_view` (projector.hpp:308),
`rasterize_backward` (projector.hpp:371), `voxelize` (voxelizer.hpp:162),
`voxelize_full` (voxelizer.hpp:203), `voxelize_backward` (voxelizer.hpp:214), plus the
helpers `view_frame`, `project_cloud`, `bin_tiles`, `sample_subvolume`,
`default_geometry` and the seeded `Rng`. Invalid input raises `ContractError`
(gsct::contract_error). Batched forms (`rasterize_views`, `rasterize_backward_views`)
process many views per call; gradients are summed over views in ascending order, exactly
`ParamGradients::add` (core.hpp:152-162).

Arrays may be numpy (host; copied in/out inside the call) or torch CUDA tensors
(device-resident; used in place). There is no CPU fallback: without the CUDA library or
a GPU every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "libgsct_b200.so"
if os.environ.get("GSCT_LIB_PATH"):  # A/B experiments with alternative builds (tools/)
    _LIB_PATH = Path(os.environ["GSCT_LIB_PATH"]).resolve()

GSCT_OK, GSCT_ERR_CONTRACT, GSCT_ERR_CUDA, GSCT_ERR_OOM, GSCT_ERR_PARSE = 0, 1, 2, 3, 4
# enum gsct_phase (include/gsct_cuda.h)
PHASES = ("raster_setup", "raster_bin", "raster_fwd", "raster_bwd", "raster_tail",
          "voxel_setup", "voxel_bin", "voxel_fwd", "voxel_bwd", "voxel_tail", "raster_order")
GSCT_HOST, GSCT_DEVICE, GSCT_HOST_ZEROED = 0, 1, 2


class GsctError(RuntimeError):
    """Base error (gsct::error)."""


class ParseError(GsctError):
    """gsct::parse_error (common.hpp:23-27); .offset = the byte offset in the message."""

    @property
    def offset(self) -> int:
        import re
        m = re.search(r"\(byte offset (\d+)\)$", str(self))
        return int(m.group(1)) if m else -1


class ContractError(GsctError):
    """Violated precondition (gsct::contract_error, common.hpp:15-17)."""


class CudaError(GsctError):
    pass


class OutOfMemoryError(CudaError):
    pass


# ---------------------------------------------------------------------------------------
# C structs (include/gsct_cuda.h)
# ---------------------------------------------------------------------------------------
class c_geometry(C.Structure):
    _fields_ = [("cone", C.c_int), ("n_u", C.c_int), ("n_v", C.c_int), ("s_u", C.c_double),
                ("s_v", C.c_double), ("source_to_origin", C.c_double), ("origin_to_detector", C.c_double)]


class c_raster_settings(C.Structure):
    _fields_ = [("tau_cut", C.c_double), ("sigma_cap", C.c_double), ("dilation_px2", C.c_double),
                ("tile_size", C.c_int), ("dilate", C.c_int), ("bounding", C.c_int)]


class c_voxel_settings(C.Structure):
    _fields_ = [("tau_cut", C.c_double), ("sigma_cap", C.c_double)]


class c_grid(C.Structure):
    _fields_ = [("dims", C.c_int * 3), ("spacing", C.c_double), ("origin", C.c_double * 3)]


class c_window(C.Structure):
    _fields_ = [("lo", C.c_int * 3), ("hi", C.c_int * 3)]


class c_stats(C.Structure):
    _fields_ = [("culled", C.c_int64), ("degenerate", C.c_int64), ("tile_pairs", C.c_int64),
                ("pixel_pairs", C.c_int64), ("forward_ms", C.c_double), ("backward_ms", C.c_double)]


class c_cloud(C.Structure):
    _fields_ = [("n", C.c_int64), ("pos", C.c_void_p), ("log_scale", C.c_void_p), ("quat", C.c_void_p),
                ("raw_density", C.c_void_p), ("location", C.c_int)]


class c_learning_rates(C.Structure):
    _fields_ = [("position", C.c_double), ("log_scale", C.c_double), ("rotation", C.c_double),
                ("density", C.c_double)]


class c_adam_state(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("m_pos", "v_pos", "m_ls", "v_ls", "m_rot", "v_rot", "m_dens", "v_dens")] + \
               [("step", C.c_int64), ("skipped_updates", C.c_int64)]


class c_control_accum(C.Structure):
    _fields_ = [("grad_norm", C.c_void_p), ("grad_dir", C.c_void_p), ("count", C.c_void_p)]


class c_rng_state(C.Structure):
    _fields_ = [("x", C.c_uint64 * 312), ("p", C.c_uint64)]


class c_control_config(C.Structure):
    _fields_ = [("grad_threshold", C.c_double), ("prune_density", C.c_double),
                ("split_scale_fraction", C.c_double), ("scene_extent", C.c_double), ("max_gaussians", C.c_int64)]


class c_adaptive_report(C.Structure):
    _fields_ = [("pruned", C.c_int64), ("cloned", C.c_int64), ("split", C.c_int64), ("n_next", C.c_int64)]


class c_grads(C.Structure):
    _fields_ = [("pos", C.c_void_p), ("log_scale", C.c_void_p), ("quat", C.c_void_p),
                ("raw_density", C.c_void_p), ("pos_grad_norm", C.c_void_p), ("visible", C.c_void_p),
                ("location", C.c_int)]


class c_group_id(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 128)]


_P = C.POINTER
_SIGS = {
    "gsct_abi_version": (C.c_int, []),
    "gsct_ctx_create": (C.c_int, [C.c_int, _P(C.c_void_p)]),
    "gsct_ctx_destroy": (None, [C.c_void_p]),
    "gsct_ctx_last_error": (C.c_char_p, [C.c_void_p]),
    "gsct_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gsct_ctx_stream": (C.c_void_p, [C.c_void_p]),
    "gsct_ctx_set_async": (C.c_int, [C.c_void_p, C.c_int]),
    "gsct_ctx_set_save_for_backward": (C.c_int, [C.c_void_p, C.c_int]),
    "gsct_ctx_synchronize": (C.c_int, [C.c_void_p, _P(c_stats)]),
    "gsct_ctx_workspace_bytes": (C.c_size_t, [C.c_void_p]),
    "gsct_ctx_launch_count": (C.c_int64, [C.c_void_p]),
    "gsct_ctx_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "gsct_ctx_phase_times": (C.c_int, [C.c_void_p, _P(C.c_double), _P(C.c_int64)]),
    "gsct_microbench": (C.c_int, [C.c_void_p, C.c_int, _P(C.c_double)]),
    "gsct_group_new_id": (C.c_int, [C.c_void_p, _P(c_group_id)]),
    "gsct_group_create": (C.c_int, [C.c_void_p, _P(c_group_id), C.c_int, C.c_int, _P(C.c_void_p)]),
    "gsct_ctx_set_group": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gsct_group_info": (C.c_int, [C.c_void_p, _P(C.c_int), _P(C.c_int)]),
    "gsct_group_destroy": (None, [C.c_void_p]),
    "gsct_rasterize_fwd": (C.c_int, [C.c_void_p, _P(c_cloud), _P(c_geometry), _P(C.c_double), C.c_int,
                                     _P(c_raster_settings), C.c_void_p, C.c_int, _P(c_stats)]),
    "gsct_rasterize_bwd": (C.c_int, [C.c_void_p, _P(c_cloud), _P(c_geometry), _P(C.c_double), C.c_int,
                                     _P(c_raster_settings), C.c_void_p, C.c_int, _P(c_grads), _P(c_stats)]),
    "gsct_voxelize_fwd": (C.c_int, [C.c_void_p, _P(c_cloud), _P(c_grid), _P(c_window), _P(c_voxel_settings),
                                    C.c_void_p, C.c_int, _P(c_stats)]),
    "gsct_voxelize_bwd": (C.c_int, [C.c_void_p, _P(c_cloud), _P(c_grid), _P(c_window), _P(c_voxel_settings),
                                    C.c_void_p, C.c_int, _P(c_grads), _P(c_stats)]),
    "gsct_voxelize_bwd_moments": (C.c_int, [C.c_void_p, _P(c_cloud), _P(c_grid), _P(c_window),
                                            _P(c_voxel_settings), C.c_void_p, C.c_int, C.c_void_p]),
    "gsct_voxelize_bwd_finish": (C.c_int, [C.c_void_p, _P(c_cloud), _P(c_grid), _P(c_voxel_settings),
                                           C.c_void_p, _P(c_grads)]),
    "gsct_debug_project": (C.c_int, [C.c_void_p, _P(c_cloud), _P(c_geometry), C.c_double, _P(c_raster_settings),
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gsct_debug_fwd_bins": (C.c_int, [C.c_void_p, _P(c_cloud), _P(c_geometry), _P(C.c_double), C.c_int,
                                      _P(c_raster_settings), C.c_void_p, C.c_void_p, C.c_int64, _P(C.c_int64)]),
    "gsct_debug_tile_pairs": (C.c_int, [C.c_void_p, _P(c_cloud), _P(c_geometry), _P(C.c_double), C.c_int,
                                        _P(c_raster_settings), C.c_void_p, C.c_void_p, C.c_int64,
                                        _P(C.c_int64)]),
    "gsct_debug_voxel_boxes": (C.c_int, [C.c_void_p, _P(c_cloud), _P(c_grid), _P(c_window),
                                         _P(c_voxel_settings), C.c_void_p, C.c_void_p, C.c_void_p]),
    "gsct_image_loss": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double,
                                  C.c_void_p, C.c_int, _P(C.c_double)]),
    "gsct_volume_loss": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, _P(C.c_int), C.c_double, C.c_void_p,
                                   C.c_int, _P(C.c_double)]),
    "gsct_tv3d": (C.c_int, [C.c_void_p, C.c_void_p, _P(C.c_int), C.c_void_p, C.c_int, _P(C.c_double)]),
    "gsct_raymarch_project": (C.c_int, [C.c_void_p, C.c_void_p, _P(c_grid), C.c_int, _P(c_geometry), _P(C.c_double),
                                        C.c_int, C.c_void_p, C.c_int]),
    "gsct_adam_step": (C.c_int, [C.c_void_p, _P(c_cloud), _P(c_adam_state), _P(c_grads), _P(c_learning_rates)]),
    "gsct_accumulate_control_stats": (C.c_int, [C.c_void_p, C.c_int64, _P(c_grads), _P(c_control_accum)]),
    "gsct_adaptive_control": (C.c_int, [C.c_void_p, _P(c_cloud), _P(c_adam_state), _P(c_control_accum),
                                        _P(c_rng_state), _P(c_control_config), C.c_int64, _P(c_cloud),
                                        _P(c_adam_state), _P(c_control_accum), _P(c_adaptive_report)]),
    "gsct_compress_model": (C.c_int, [C.c_void_p, _P(c_cloud), C.c_void_p, C.c_int, _P(C.c_int64)]),
    "gsct_decompress_model": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, _P(c_cloud)]),
    "gsct_host_view_frame": (None, [_P(c_geometry), C.c_double, _P(C.c_double)]),
    "gsct_host_default_geometry": (None, [_P(C.c_int), C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                          _P(c_geometry), _P(C.c_double)]),
    "gsct_host_rng_create": (C.c_void_p, [C.c_uint64]),
    "gsct_host_rng_destroy": (None, [C.c_void_p]),
    "gsct_host_rng_uniform": (C.c_double, [C.c_void_p, C.c_double, C.c_double]),
    "gsct_host_rng_normal": (C.c_double, [C.c_void_p]),
    "gsct_host_rng_uniform_int": (C.c_int64, [C.c_void_p, C.c_int64]),
    "gsct_host_rng_get_state": (None, [C.c_void_p, _P(c_rng_state)]),
    "gsct_host_rng_set_state": (None, [C.c_void_p, _P(c_rng_state)]),
    "gsct_host_sample_subvolume": (C.c_int, [_P(C.c_int), _P(C.c_int), C.c_void_p, _P(C.c_int), _P(C.c_int)]),
    "gsct_host_f64_to_f32": (None, [C.c_void_p, C.c_void_p, C.c_int64]),
    "gsct_host_f32_to_f64": (None, [C.c_void_p, C.c_void_p, C.c_int64, C.c_double]),
    "gsct_host_make_cloud": (C.c_int, [C.c_int, C.c_int64, C.c_uint64, _P(C.c_double), C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p]),
}

_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Loads libgsct_b200.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(f"{_LIB_PATH} is missing: run `python -m paper_2604_01844_b200.build_native` "
                              "(there is no CPU fallback)")
        l = C.CDLL(str(_LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


# ---------------------------------------------------------------------------------------
# Reference-mirroring value types
# ---------------------------------------------------------------------------------------
@dataclass
class ScanGeometry:
    """gsct::ScanGeometry (core.hpp:203-222)."""
    mode: str = "parallel"  # "parallel" | "cone"
    n_u: int = 0
    n_v: int = 0
    s_u: float = 1.0
    s_v: float = 1.0
    angles: Sequence[float] = field(default_factory=list)
    source_to_origin: float = 0.0
    origin_to_detector: float = 0.0

    def n_views(self) -> int:
        return len(self.angles)

    def c(self) -> c_geometry:
        if self.mode not in ("parallel", "cone"):
            raise ContractError(f"ScanGeometry: unknown mode {self.mode!r}")
        return c_geometry(1 if self.mode == "cone" else 0, int(self.n_u), int(self.n_v), float(self.s_u),
                          float(self.s_v), float(self.source_to_origin), float(self.origin_to_detector))


@dataclass
class RasterSettings:
    """gsct::RasterSettings (projector.hpp:64-71)."""
    tau_cut: float = 1e-4
    sigma_cap: float = 3.0
    tile_size: int = 16
    dilate: bool = True
    dilation_px2: float = 0.3
    bounding: str = "rect_density_aware"  # | "square_circumscribed"

    def c(self) -> c_raster_settings:
        return c_raster_settings(float(self.tau_cut), float(self.sigma_cap), float(self.dilation_px2),
                                 int(self.tile_size), 1 if self.dilate else 0,
                                 1 if self.bounding == "square_circumscribed" else 0)


@dataclass
class VoxelSettings:
    """gsct::VoxelSettings (voxelizer.hpp:99-102)."""
    tau_cut: float = 1e-4
    sigma_cap: float = 3.0

    def c(self) -> c_voxel_settings:
        return c_voxel_settings(float(self.tau_cut), float(self.sigma_cap))


@dataclass
class RenderStats:
    """gsct::RenderStats (projector.hpp:73-80), accumulated with +=."""
    culled: int = 0
    degenerate: int = 0
    tile_pairs: int = 0
    pixel_pairs: int = 0
    forward_ms: float = 0.0
    backward_ms: float = 0.0

    def _c(self) -> c_stats:
        return c_stats(self.culled, self.degenerate, self.tile_pairs, self.pixel_pairs, self.forward_ms,
                       self.backward_ms)

    def _take(self, s: c_stats) -> None:
        self.culled, self.degenerate = s.culled, s.degenerate
        self.tile_pairs, self.pixel_pairs = s.tile_pairs, s.pixel_pairs
        self.forward_ms, self.backward_ms = s.forward_ms, s.backward_ms


@dataclass
class GridSpec:
    """gsct::GridSpec (voxelizer.hpp:22-41)."""
    dims: tuple = (0, 0, 0)
    spacing: float = 1.0
    origin: tuple = (0.0, 0.0, 0.0)

    @staticmethod
    def centered(dims, spacing: float) -> "GridSpec":
        return GridSpec(tuple(int(d) for d in dims), float(spacing),
                        tuple(-0.5 * spacing * (d - 1) for d in dims))

    def count(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])


@dataclass
class GridRegion:
    """gsct::GridRegion (voxelizer.hpp:43-71)."""
    offset: tuple = (0, 0, 0)
    dims: tuple = (0, 0, 0)
    spacing: float = 1.0
    origin: tuple = (0.0, 0.0, 0.0)

    @staticmethod
    def covering(parent: GridSpec) -> "GridRegion":
        return GridRegion((0, 0, 0), tuple(parent.dims), parent.spacing, tuple(parent.origin))

    @staticmethod
    def of_parent(parent: GridSpec, offset, dims) -> "GridRegion":
        for a in range(3):
            if not dims[a] >= 1:
                raise ContractError("GridRegion: dims must be at least 1")
            if not (offset[a] >= 0 and offset[a] + dims[a] <= parent.dims[a]):
                raise ContractError("GridRegion: region outside parent grid")
        origin = tuple(parent.origin[a] + parent.spacing * float(offset[a]) for a in range(3))
        return GridRegion(tuple(int(o) for o in offset), tuple(int(d) for d in dims), parent.spacing, origin)

    def count(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class GaussianCloud:
    """gsct::GaussianCloud (core.hpp:30-59): raw parameters, AoS doubles.

    Holds numpy float64 arrays (host) or torch float64 CUDA tensors (device-resident).
    """

    def __init__(self, positions, log_scales, rotations, raw_densities):
        self.positions = positions
        self.log_scales = log_scales
        self.rotations = rotations
        self.raw_densities = raw_densities
        self.validate()

    @staticmethod
    def empty() -> "GaussianCloud":
        return GaussianCloud(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0,)))

    def size(self) -> int:
        return int(self.positions.shape[0])

    def __len__(self) -> int:
        return self.size()

    def validate(self) -> None:
        n = self.positions.shape[0]
        if not (self.log_scales.shape[0] == n and self.rotations.shape[0] == n and self.raw_densities.shape[0] == n):
            raise ContractError("GaussianCloud: parameter arrays out of lockstep")

    @property
    def on_device(self) -> bool:
        return _is_torch(self.positions) and self.positions.is_cuda

    def to_device(self, device: int = 0) -> "GaussianCloud":
        import torch
        f = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(f"cuda:{device}")
        return GaussianCloud(f(self.positions), f(self.log_scales), f(self.rotations), f(self.raw_densities))

    def numpy(self) -> "GaussianCloud":
        if not _is_torch(self.positions):
            return self
        f = lambda a: a.detach().cpu().numpy()
        return GaussianCloud(f(self.positions), f(self.log_scales), f(self.rotations), f(self.raw_densities))

    def _c(self, keep: list) -> c_cloud:
        self.validate()
        n = self.size()
        if self.on_device:
            arrs = [self.positions, self.log_scales, self.rotations, self.raw_densities]
            for a in arrs:
                if a.dtype != __import__("torch").float64 or not a.is_contiguous():
                    raise ContractError("GaussianCloud: device arrays must be contiguous float64")
            keep.extend(arrs)
            return c_cloud(n, arrs[0].data_ptr(), arrs[1].data_ptr(), arrs[2].data_ptr(), arrs[3].data_ptr(),
                           GSCT_DEVICE)
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (self.positions, self.log_scales, self.rotations, self.raw_densities)]
        keep.extend(arrs)
        ptr = lambda a: a.ctypes.data if a.size else None
        return c_cloud(n, ptr(arrs[0]), ptr(arrs[1]), ptr(arrs[2]), ptr(arrs[3]), GSCT_HOST)


@dataclass
class ParamGradients:
    """gsct::ParamGradients (core.hpp:135-163)."""
    positions: object
    log_scales: object
    rotations: object
    raw_densities: object
    pos_grad_norm: object
    visible: object

    @staticmethod
    def zeros(n: int, device: Optional[int] = None) -> "ParamGradients":
        if device is None:
            z = lambda *s: np.zeros(s, dtype=np.float64)
            return ParamGradients(z(n, 3), z(n, 3), z(n, 4), z(n), z(n), np.zeros(n, dtype=np.uint8))
        import torch
        z = lambda *s: torch.zeros(s, dtype=torch.float64, device=f"cuda:{device}")
        return ParamGradients(z(n, 3), z(n, 3), z(n, 4), z(n), z(n),
                              torch.zeros(n, dtype=torch.uint8, device=f"cuda:{device}"))

    def add(self, other: "ParamGradients") -> None:
        """ParamGradients::add (core.hpp:152-162)."""
        if other.positions.shape[0] != self.positions.shape[0]:
            raise ContractError("ParamGradients::add: size mismatch")
        self.positions = self.positions + other.positions
        self.log_scales = self.log_scales + other.log_scales
        self.rotations = self.rotations + other.rotations
        self.raw_densities = self.raw_densities + other.raw_densities
        self.pos_grad_norm = self.pos_grad_norm + other.pos_grad_norm
        self.visible = self.visible | other.visible

    def _c(self, zeroed: bool = False) -> c_grads:
        """zeroed: host arrays known to be zero-filled (GSCT_HOST_ZEROED: sparse outputs may skip rows)."""
        arrs = [self.positions, self.log_scales, self.rotations, self.raw_densities, self.pos_grad_norm, self.visible]
        if _is_torch(self.positions):
            return c_grads(*[a.data_ptr() for a in arrs], GSCT_DEVICE)
        return c_grads(*[a.ctypes.data if a.size else None for a in arrs], GSCT_HOST_ZEROED if zeroed else GSCT_HOST)


# ---------------------------------------------------------------------------------------
# Context (one per CUDA device)
# ---------------------------------------------------------------------------------------
class Context:
    """Owns a gsct_ctx: stream, grow-only device workspace, last error."""

    def __init__(self, device: int = 0):
        self._lib = lib()
        h = C.c_void_p()
        st = self._lib.gsct_ctx_create(int(device), C.byref(h))
        if st != GSCT_OK:
            raise CudaError(f"gsct_ctx_create(device={device}) failed: no usable CUDA device "
                            "(libgsct_b200 has no CPU fallback)")
        self.handle = h
        self.device = int(device)

    def close(self) -> None:
        if getattr(self, "handle", None):
            self._lib.gsct_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, status: int) -> None:
        if status == GSCT_OK:
            return
        msg = self._lib.gsct_ctx_last_error(self.handle).decode(errors="replace")
        if status == GSCT_ERR_CONTRACT:
            raise ContractError(msg)
        if status == GSCT_ERR_OOM:
            raise OutOfMemoryError(msg)
        if status == GSCT_ERR_PARSE:
            raise ParseError(msg)
        raise CudaError(msg)

    def set_stream(self, stream_ptr: int) -> None:
        self.check(self._lib.gsct_ctx_set_stream(self.handle, C.c_void_p(stream_ptr)))

    def set_async(self, on: bool) -> None:
        self.check(self._lib.gsct_ctx_set_async(self.handle, 1 if on else 0))

    def set_save_for_backward(self, on: bool) -> None:
        """Keep the forward's set-up for the matching backward (caller keeps the cloud fixed)."""
        self.check(self._lib.gsct_ctx_set_save_for_backward(self.handle, 1 if on else 0))

    def synchronize(self, stats: Optional[RenderStats] = None) -> None:
        s = stats._c() if stats is not None else c_stats()
        self.check(self._lib.gsct_ctx_synchronize(self.handle, C.byref(s)))
        if stats is not None:
            stats._take(s)

    def launch_count(self) -> int:
        return int(self._lib.gsct_ctx_launch_count(self.handle))

    def workspace_bytes(self) -> int:
        return int(self._lib.gsct_ctx_workspace_bytes(self.handle))

    def set_profiling(self, on: bool) -> None:
        self.check(self._lib.gsct_ctx_set_profiling(self.handle, 1 if on else 0))

    def phase_times(self) -> dict:
        """Accumulated device ms and launch counts per phase since the last call."""
        ms = (C.c_double * len(PHASES))()
        cnt = (C.c_int64 * len(PHASES))()
        self.check(self._lib.gsct_ctx_phase_times(self.handle, ms, cnt))
        return {name: (ms[i], cnt[i]) for i, name in enumerate(PHASES)}

    def group_new_id(self) -> bytes:
        """A fresh 128-byte group id (ncclUniqueId); rank 0 makes it, every rank gets a copy."""
        gid = c_group_id()
        self.check(self._lib.gsct_group_new_id(self.handle, C.byref(gid)))
        return bytes(gid.bytes)

    def create_group(self, group_id: bytes, n_ranks: int, rank: int, attach: bool = True) -> "Group":
        """Collective over all ranks: the NCCL communicator of this context's device. With
        attach, the backward / voxel calls of this context run their cross-rank reductions
        (include/gsct_cuda.h, multi-GPU)."""
        if len(group_id) != 128:
            raise ContractError("gsct_group_create: the group id is 128 bytes")
        gid = c_group_id()
        C.memmove(gid.bytes, group_id, 128)
        h = C.c_void_p()
        self.check(self._lib.gsct_group_create(self.handle, C.byref(gid), int(n_ranks), int(rank), C.byref(h)))
        g = Group(self._lib, h)
        if attach:
            self.set_group(g)
        return g

    def set_group(self, group: Optional["Group"]) -> None:
        self.check(self._lib.gsct_ctx_set_group(self.handle, group.handle if group is not None else None))
        self._group = group

    def microbench(self, kind: str) -> float:
        """Device-wide ops/s: "ex2" (MUFU ex2.approx.f32) or "ffma" (FP32 FFMA)."""
        out = C.c_double(0.0)
        self.check(self._lib.gsct_microbench(self.handle, {"ex2": 0, "ffma": 1}[kind], C.byref(out)))
        return out.value


class Group:
    """A gsct_group (one NCCL communicator per context)."""

    def __init__(self, lib_, handle):
        self._lib = lib_
        self.handle = handle
        r, n = C.c_int(0), C.c_int(0)
        lib_.gsct_group_info(handle, C.byref(r), C.byref(n))
        self.rank, self.size = r.value, n.value

    def close(self) -> None:
        if getattr(self, "handle", None):
            self._lib.gsct_group_destroy(self.handle)
            self.handle = None


_contexts: dict[int, Context] = {}


def context(device: int = 0) -> Context:
    if device not in _contexts:
        _contexts[device] = Context(device)
    return _contexts[device]


def _ptr(x, keep: list):
    """(pointer, location) for a numpy array or torch CUDA tensor."""
    if _is_torch(x):
        if not x.is_cuda:
            x = x.contiguous()
            keep.append(x)
            return x.data_ptr(), GSCT_HOST
        if not x.is_contiguous():
            raise ContractError("device buffers must be contiguous")
        keep.append(x)
        return x.data_ptr(), GSCT_DEVICE
    keep.append(x)
    return x.ctypes.data, GSCT_HOST


def _ctx_for(cloud: GaussianCloud, ctx: Optional[Context]) -> Context:
    if ctx is not None:
        return ctx
    dev = cloud.positions.device.index if cloud.on_device else 0
    return context(dev or 0)


def _angles(geometry: ScanGeometry, view_indices) -> np.ndarray:
    angles = np.asarray(geometry.angles, dtype=np.float64)
    if view_indices is None:
        return np.ascontiguousarray(angles)
    idx = np.asarray(view_indices, dtype=np.int64).reshape(-1)
    if idx.size and (idx.min() < 0 or idx.max() >= angles.size):
        raise ContractError("view_frame: angle index out of range")
    return np.ascontiguousarray(angles[idx])


# ---------------------------------------------------------------------------------------
# Rasterizer (projector.hpp)
# ---------------------------------------------------------------------------------------
def rasterize_views(cloud: GaussianCloud, geometry: ScanGeometry, view_indices=None,
                    settings: RasterSettings = RasterSettings(), stats: Optional[RenderStats] = None,
                    out=None, ctx: Optional[Context] = None):
    """Forward projection of several views: images [V, n_v, n_u] float32 (u fastest)."""
    ctx = _ctx_for(cloud, ctx)
    ang = _angles(geometry, view_indices)
    keep: list = []
    cc = cloud._c(keep)
    if out is None:
        if cloud.on_device:
            import torch
            out = torch.empty((ang.size, geometry.n_v, geometry.n_u), dtype=torch.float32,
                              device=cloud.positions.device)
        else:
            out = np.empty((ang.size, geometry.n_v, geometry.n_u), dtype=np.float32)
    optr, oloc = _ptr(out, keep)
    s = stats._c() if stats is not None else c_stats()
    g = geometry.c()
    rs = settings.c()
    ctx.check(ctx._lib.gsct_rasterize_fwd(ctx.handle, C.byref(cc), C.byref(g),
                                          ang.ctypes.data_as(_P(C.c_double)), int(ang.size), C.byref(rs),
                                          C.c_void_p(optr), oloc, C.byref(s) if stats is not None else None))
    if stats is not None:
        stats._take(s)
    return out


def rasterize_view(cloud: GaussianCloud, geometry: ScanGeometry, angle_index: int,
                   settings: RasterSettings = RasterSettings(), stats: Optional[RenderStats] = None,
                   ctx: Optional[Context] = None):
    """gsct::rasterize_view: one view, image [n_v, n_u] float32."""
    return rasterize_views(cloud, geometry, [angle_index], settings, stats, ctx=ctx)[0]


def rasterize_backward_views(cloud: GaussianCloud, geometry: ScanGeometry, view_indices, grad_images,
                             settings: RasterSettings = RasterSettings(), stats: Optional[RenderStats] = None,
                             out: Optional[ParamGradients] = None, ctx: Optional[Context] = None) -> ParamGradients:
    """Sum over views (ascending) of rasterize_backward; grad_images [V, n_v, n_u] float32."""
    ctx = _ctx_for(cloud, ctx)
    ang = _angles(geometry, view_indices)
    shape = tuple(grad_images.shape)
    if shape != (ang.size, geometry.n_v, geometry.n_u):
        raise ContractError("rasterize_backward: grad image dims must match detector")
    keep: list = []
    cc = cloud._c(keep)
    if _is_torch(grad_images):
        import torch
        if grad_images.dtype != torch.float32:
            grad_images = grad_images.float()
    else:
        grad_images = np.ascontiguousarray(grad_images, dtype=np.float32)
    gptr, gloc = _ptr(grad_images, keep)
    if out is None:
        out = ParamGradients.zeros(cloud.size(), cloud.positions.device.index if cloud.on_device else None)
    cg = out._c()
    s = stats._c() if stats is not None else c_stats()
    g = geometry.c()
    rs = settings.c()
    ctx.check(ctx._lib.gsct_rasterize_bwd(ctx.handle, C.byref(cc), C.byref(g), ang.ctypes.data_as(_P(C.c_double)),
                                          int(ang.size), C.byref(rs), C.c_void_p(gptr), gloc, C.byref(cg),
                                          C.byref(s) if stats is not None else None))
    if stats is not None:
        stats._take(s)
    return out


def rasterize_backward(cloud: GaussianCloud, geometry: ScanGeometry, angle_index: int, grad_image,
                       settings: RasterSettings = RasterSettings(), stats: Optional[RenderStats] = None,
                       ctx: Optional[Context] = None) -> ParamGradients:
    """gsct::rasterize_backward for one view."""
    if tuple(grad_image.shape) != (geometry.n_v, geometry.n_u):
        raise ContractError("rasterize_backward: grad image dims must match detector")
    return rasterize_backward_views(cloud, geometry, [angle_index], grad_image[None], settings, stats, ctx=ctx)


# ---------------------------------------------------------------------------------------
# Voxelizer (voxelizer.hpp)
# ---------------------------------------------------------------------------------------
def _grid_c(region) -> c_grid:
    return c_grid((C.c_int * 3)(*[int(d) for d in region.dims]), float(region.spacing),
                  (C.c_double * 3)(*[float(o) for o in region.origin]))


def _window_c(window) -> Optional[c_window]:
    if window is None:
        return None
    lo, hi = window
    return c_window((C.c_int * 3)(*[int(v) for v in lo]), (C.c_int * 3)(*[int(v) for v in hi]))


def voxelize(cloud: GaussianCloud, region, settings: VoxelSettings = VoxelSettings(),
             stats: Optional[RenderStats] = None, window=None, out=None, ctx: Optional[Context] = None):
    """gsct::voxelize: volume [nz, ny, nx] float32 (x fastest). `window` = ((x0,y0,z0),(x1,y1,z1))
    restricts the output to a sub-box of the region (z-slab sharding) without changing values."""
    ctx = _ctx_for(cloud, ctx)
    keep: list = []
    cc = cloud._c(keep)
    gr = _grid_c(region)
    win = _window_c(window)
    lo, hi = window if window is not None else ((0, 0, 0), tuple(region.dims))
    shape = (hi[2] - lo[2], hi[1] - lo[1], hi[0] - lo[0])
    if out is None:
        if cloud.on_device:
            import torch
            out = torch.empty(shape, dtype=torch.float32, device=cloud.positions.device)
        else:
            out = np.empty(shape, dtype=np.float32)
    optr, oloc = _ptr(out, keep)
    s = stats._c() if stats is not None else c_stats()
    vs = settings.c()
    ctx.check(ctx._lib.gsct_voxelize_fwd(ctx.handle, C.byref(cc), C.byref(gr), C.byref(win) if win else None,
                                         C.byref(vs), C.c_void_p(optr), oloc,
                                         C.byref(s) if stats is not None else None))
    if stats is not None:
        stats._take(s)
    return out


def voxelize_full(cloud: GaussianCloud, grid: GridSpec, settings: VoxelSettings = VoxelSettings(),
                  stats: Optional[RenderStats] = None, ctx: Optional[Context] = None):
    """gsct::voxelize_full (voxelizer.hpp:203-206)."""
    return voxelize(cloud, GridRegion.covering(grid), settings, stats, ctx=ctx)


def voxelize_backward(cloud: GaussianCloud, region, grad_volume, settings: VoxelSettings = VoxelSettings(),
                      stats: Optional[RenderStats] = None, out: Optional[ParamGradients] = None,
                      ctx: Optional[Context] = None) -> ParamGradients:
    """gsct::voxelize_backward; grad_volume [nz, ny, nx] float32."""
    if tuple(grad_volume.shape) != (region.dims[2], region.dims[1], region.dims[0]):
        raise ContractError("voxelize_backward: grad dims must match region")
    ctx = _ctx_for(cloud, ctx)
    keep: list = []
    cc = cloud._c(keep)
    if _is_torch(grad_volume):
        grad_volume = grad_volume.float().contiguous()
    else:
        grad_volume = np.ascontiguousarray(grad_volume, dtype=np.float32)
    gptr, gloc = _ptr(grad_volume, keep)
    fresh = out is None  # zero-filled here: the library may transfer only the touched splats' rows
    if out is None:
        out = ParamGradients.zeros(cloud.size(), cloud.positions.device.index if cloud.on_device else None)
    cg = out._c(zeroed=fresh)
    s = stats._c() if stats is not None else c_stats()
    gr = _grid_c(region)
    vs = settings.c()
    ctx.check(ctx._lib.gsct_voxelize_bwd(ctx.handle, C.byref(cc), C.byref(gr), None, C.byref(vs), C.c_void_p(gptr),
                                         gloc, C.byref(cg), C.byref(s) if stats is not None else None))
    if stats is not None:
        stats._take(s)
    return out


def voxelize_backward_moments(cloud: GaussianCloud, region, grad_window, window, moments,
                              settings: VoxelSettings = VoxelSettings(), ctx: Optional[Context] = None):
    """Per-splat partial sums over one window (z-slab) into device moments [10, N] float64
    (each splat's window sum formed in fp32, then widened; reduced across ranks in fp64)."""
    ctx = _ctx_for(cloud, ctx)
    keep: list = []
    cc = cloud._c(keep)
    gptr, gloc = _ptr(grad_window, keep)
    mptr, mloc = _ptr(moments, keep)
    if mloc != GSCT_DEVICE or str(moments.dtype) != "torch.float64" or tuple(moments.shape) != (10, cloud.size()):
        raise ContractError("voxelize_backward_moments: moments must be a [10, N] float64 CUDA tensor")
    gr = _grid_c(region)
    win = _window_c(window)
    vs = settings.c()
    ctx.check(ctx._lib.gsct_voxelize_bwd_moments(ctx.handle, C.byref(cc), C.byref(gr), C.byref(win) if win else None,
                                                 C.byref(vs), C.c_void_p(gptr), gloc, C.c_void_p(mptr)))
    return moments


def voxelize_backward_finish(cloud: GaussianCloud, region, moments, settings: VoxelSettings = VoxelSettings(),
                             out: Optional[ParamGradients] = None, ctx: Optional[Context] = None) -> ParamGradients:
    ctx = _ctx_for(cloud, ctx)
    keep: list = []
    cc = cloud._c(keep)
    mptr, _ = _ptr(moments, keep)
    if out is None:
        out = ParamGradients.zeros(cloud.size(), cloud.positions.device.index if cloud.on_device else None)
    cg = out._c()
    gr = _grid_c(region)
    vs = settings.c()
    ctx.check(ctx._lib.gsct_voxelize_bwd_finish(ctx.handle, C.byref(cc), C.byref(gr), C.byref(vs), C.c_void_p(mptr),
                                                C.byref(cg)))
    return out


# ---------------------------------------------------------------------------------------
# Parity hooks and helpers
# ---------------------------------------------------------------------------------------
def project_cloud(cloud: GaussianCloud, geometry: ScanGeometry, angle_index: int,
                  settings: RasterSettings = RasterSettings(), ctx: Optional[Context] = None) -> dict:
    """gsct::project_cloud on the device: per-splat rect [N,4], culled, degenerate, mean2d, conic, amplitude."""
    ctx = _ctx_for(cloud, ctx)
    keep: list = []
    cc = cloud._c(keep)
    n = cloud.size()
    rect = np.zeros((n, 4), dtype=np.int32)
    flags = np.zeros(n, dtype=np.uint8)
    mean2d = np.zeros((n, 2))
    conic = np.zeros((n, 4))
    amp = np.zeros(n)
    theta = float(_angles(geometry, [angle_index])[0])
    g = geometry.c()
    rs = settings.c()
    ctx.check(ctx._lib.gsct_debug_project(ctx.handle, C.byref(cc), C.byref(g), theta, C.byref(rs),
                                          rect.ctypes.data, flags.ctypes.data, mean2d.ctypes.data,
                                          conic.ctypes.data, amp.ctypes.data))
    return dict(rect=rect, culled=(flags & 1).astype(bool), degenerate=(flags & 2).astype(bool), mean2d=mean2d,
                conic=conic, amplitude=amp)


def tile_pairs(cloud: GaussianCloud, geometry: ScanGeometry, view_indices=None,
               settings: RasterSettings = RasterSettings(), ctx: Optional[Context] = None):
    """Sorted (key, splat) pairs of the device binning (key = view*n_tiles + tile)."""
    ctx = _ctx_for(cloud, ctx)
    ang = _angles(geometry, view_indices)
    keep: list = []
    cc = cloud._c(keep)
    g = geometry.c()
    rs = settings.c()
    n_pairs = C.c_int64(0)
    ctx.check(ctx._lib.gsct_debug_tile_pairs(ctx.handle, C.byref(cc), C.byref(g), ang.ctypes.data_as(_P(C.c_double)),
                                             int(ang.size), C.byref(rs), None, None, 0, C.byref(n_pairs)))
    keys = np.zeros(max(n_pairs.value, 1), dtype=np.uint32)
    vals = np.zeros(max(n_pairs.value, 1), dtype=np.uint32)
    ctx.check(ctx._lib.gsct_debug_tile_pairs(ctx.handle, C.byref(cc), C.byref(g), ang.ctypes.data_as(_P(C.c_double)),
                                             int(ang.size), C.byref(rs), keys.ctypes.data, vals.ctypes.data,
                                             n_pairs.value, C.byref(n_pairs)))
    return keys[: n_pairs.value], vals[: n_pairs.value]


def forward_bins(cloud: GaussianCloud, geometry: ScanGeometry, view_indices=None,
                 settings: RasterSettings = RasterSettings(), ctx: Optional[Context] = None):
    """The forward's own binning (gsct_debug_fwd_bins): CSR offsets over (view, 32x32
    super-tile), view-major, and the ascending splat lists. Equals bin_tiles at tile_size 32
    (projector.hpp:266-286) per view."""
    ctx = _ctx_for(cloud, ctx)
    ang = _angles(geometry, view_indices)
    keep: list = []
    cc = cloud._c(keep)
    g = geometry.c()
    rs = settings.c()
    n_st = ((geometry.n_u + 31) // 32) * ((geometry.n_v + 31) // 32)
    offsets = np.zeros(int(ang.size) * n_st + 1, dtype=np.int64)
    n_pairs = C.c_int64(0)
    ctx.check(ctx._lib.gsct_debug_fwd_bins(ctx.handle, C.byref(cc), C.byref(g), ang.ctypes.data_as(_P(C.c_double)),
                                           int(ang.size), C.byref(rs), offsets.ctypes.data, None, 0,
                                           C.byref(n_pairs)))
    splats = np.zeros(max(n_pairs.value, 1), dtype=np.uint32)
    ctx.check(ctx._lib.gsct_debug_fwd_bins(ctx.handle, C.byref(cc), C.byref(g), ang.ctypes.data_as(_P(C.c_double)),
                                           int(ang.size), C.byref(rs), offsets.ctypes.data, splats.ctypes.data,
                                           n_pairs.value, C.byref(n_pairs)))
    return offsets, splats[: n_pairs.value]


def bin_tiles(cloud: GaussianCloud, geometry: ScanGeometry, angle_index: int,
              settings: RasterSettings = RasterSettings(), ctx: Optional[Context] = None) -> list:
    """gsct::bin_tiles equivalent: per-tile ascending splat lists for one view."""
    keys, vals = tile_pairs(cloud, geometry, [angle_index], settings, ctx)
    ts = settings.tile_size
    n_tiles = ((geometry.n_u + ts - 1) // ts) * ((geometry.n_v + ts - 1) // ts)
    bins: list = [[] for _ in range(n_tiles)]
    bounds = np.searchsorted(keys, np.arange(n_tiles + 1))
    for t in range(n_tiles):
        bins[t] = vals[bounds[t]:bounds[t + 1]].astype(np.int32).tolist()
    return bins


def voxel_boxes(cloud: GaussianCloud, region, settings: VoxelSettings = VoxelSettings(), window=None,
                ctx: Optional[Context] = None):
    """detail::prepare_voxel_splats boxes on the device: lo [N,3], hi [N,3], skip [N]."""
    ctx = _ctx_for(cloud, ctx)
    keep: list = []
    cc = cloud._c(keep)
    n = cloud.size()
    lo = np.zeros((n, 3), dtype=np.int32)
    hi = np.zeros((n, 3), dtype=np.int32)
    skip = np.zeros(n, dtype=np.uint8)
    gr = _grid_c(region)
    win = _window_c(window)
    vs = settings.c()
    ctx.check(ctx._lib.gsct_debug_voxel_boxes(ctx.handle, C.byref(cc), C.byref(gr), C.byref(win) if win else None,
                                              C.byref(vs), lo.ctypes.data, hi.ctypes.data, skip.ctypes.data))
    return lo, hi, skip.astype(bool)


# ---------------------------------------------------------------------------------------
# Host-side harness (no GPU needed)
# ---------------------------------------------------------------------------------------
def view_frame(geometry: ScanGeometry, angle_index: int) -> dict:
    """gsct::view_frame (projector.hpp:29-43)."""
    theta = float(_angles(geometry, [angle_index])[0])
    f = (C.c_double * 16)()
    g = geometry.c()
    lib().gsct_host_view_frame(C.byref(g), theta, f)
    a = np.array(f[:])
    return dict(u=a[0:3], v=a[3:6], d=a[6:9], detector_center=a[9:12], source=a[12:15], focal=a[15],
                cone=geometry.mode == "cone")


def default_geometry(dims, spacing: float, n_views: int, mode: str, n_u: int, n_v: int) -> ScanGeometry:
    """gsct::default_geometry (synthetic.hpp:246-271) for a volume of `dims` at `spacing`."""
    g = c_geometry()
    angles = (C.c_double * max(n_views, 1))()
    lib().gsct_host_default_geometry((C.c_int * 3)(*[int(d) for d in dims]), float(spacing), int(n_views),
                                     1 if mode == "cone" else 0, int(n_u), int(n_v), C.byref(g), angles)
    return ScanGeometry(mode, g.n_u, g.n_v, g.s_u, g.s_v, list(angles[:n_views]), g.source_to_origin,
                        g.origin_to_detector)


class Rng:
    """gsct::Rng (rng.hpp:18-69): mt19937_64 with the reference's output mappings."""

    def __init__(self, seed: int = 0):
        self._lib = lib()
        self._h = self._lib.gsct_host_rng_create(C.c_uint64(seed))

    def __del__(self):
        try:
            self._lib.gsct_host_rng_destroy(self._h)
        except Exception:
            pass

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        return self._lib.gsct_host_rng_uniform(self._h, lo, hi)

    def normal(self) -> float:
        return self._lib.gsct_host_rng_normal(self._h)

    def uniform_int(self, n: int) -> int:
        if n <= 0:
            raise ContractError("Rng::uniform_int: n must be positive")
        return int(self._lib.gsct_host_rng_uniform_int(self._h, n))

    def uniform_array(self, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        return np.array([self.uniform(lo, hi) for _ in range(n)])

    def state(self) -> c_rng_state:
        """The engine state (Rng::save_state's numbers: x[0..311], p)."""
        st = c_rng_state()
        self._lib.gsct_host_rng_get_state(self._h, C.byref(st))
        return st

    def set_state(self, st: c_rng_state) -> None:
        self._lib.gsct_host_rng_set_state(self._h, C.byref(st))


def sample_subvolume(parent: GridSpec, sub_dims, rng: Rng) -> GridRegion:
    """gsct::sample_subvolume (voxelizer.hpp:76-93)."""
    off = (C.c_int * 3)()
    dims = (C.c_int * 3)()
    st = lib().gsct_host_sample_subvolume((C.c_int * 3)(*[int(d) for d in parent.dims]),
                                          (C.c_int * 3)(*[int(d) for d in sub_dims]), rng._h, off, dims)
    if st != 0:
        raise ContractError("sample_subvolume: dims must be at least 1")
    return GridRegion.of_parent(parent, tuple(off), tuple(dims))


def make_cloud(kind: str, count: int, seed: int = 0, **kw) -> GaussianCloud:
    """Seeded clouds: "synthetic" (bench.hpp:33-52), "random" (tests/oracles.hpp:168-184),
    "shepp_logan" (SURVEY.md 8d benchmark phantom cloud)."""
    if kind == "synthetic":
        k, p = 0, [kw.get("half_extent", 0.8), kw.get("scale", 0.04), kw.get("anisotropy", 1.0),
                   kw.get("density", 1.0)]
    elif kind == "random":
        k, p = 1, [kw.get("pos_range", 5.0), kw.get("scale_lo", 0.5), kw.get("scale_hi", 2.5)]
    elif kind == "shepp_logan":
        k, p = 2, [float(kw["side"]), float(kw.get("spacing", 1.0))]
    else:
        raise ContractError(f"make_cloud: unknown kind {kind!r}")
    pos = np.zeros((count, 3))
    ls = np.zeros((count, 3))
    q = np.zeros((count, 4))
    raw = np.zeros(count)
    pa = (C.c_double * 4)(*(p + [0.0] * (4 - len(p))))
    st = lib().gsct_host_make_cloud(k, int(count), C.c_uint64(seed), pa, pos.ctypes.data, ls.ctypes.data,
                                    q.ctypes.data, raw.ctypes.data)
    if st != 0:
        raise ContractError("make_cloud failed")
    return GaussianCloud(pos, ls, q, raw)


# ---------------------------------------------------------------------------------------
# Next-row operators: image loss, Adam
# ---------------------------------------------------------------------------------------
def image_loss(rendered, measured, alpha_ssim: float = 0.25, grad_out=None, ctx: Optional[Context] = None):
    """total_loss_recon (losses.hpp:613-637) with alpha_tv = 0, per view, on [V, n_v, n_u]
    float32 images (numpy or CUDA tensors). Returns (losses [V, 3] = {l1, ssim, total},
    grad [V, n_v, n_u] float32 = d total / d rendered, same kind as the inputs)."""
    if tuple(rendered.shape) != tuple(measured.shape) or len(rendered.shape) not in (2, 3):
        raise ContractError("l1: image shape mismatch")
    shape = tuple(rendered.shape)
    nv_, nv, nu = (1,) + shape if len(shape) == 2 else shape
    keep: list = []
    dev = _is_torch(rendered) and rendered.is_cuda
    if ctx is None:
        ctx = context(rendered.device.index or 0) if dev else context(0)
    if grad_out is None:
        if dev:
            import torch
            grad_out = torch.empty(shape, dtype=torch.float32, device=rendered.device)
        else:
            grad_out = np.empty(shape, dtype=np.float32)
    rp, rl = _ptr(rendered if dev else np.ascontiguousarray(rendered, dtype=np.float32), keep)
    mp, ml = _ptr(measured if dev else np.ascontiguousarray(measured, dtype=np.float32), keep)
    gp, gl = _ptr(grad_out, keep)
    if not (rl == ml == gl):
        raise ContractError("image_loss: rendered, measured and grad must share one location")
    losses = np.zeros((nv_, 3), dtype=np.float64)
    ctx.check(ctx._lib.gsct_image_loss(ctx.handle, C.c_void_p(rp), C.c_void_p(mp), nv_, nu, nv, float(alpha_ssim),
                                       C.c_void_p(gp), rl, losses.ctypes.data_as(C.POINTER(C.c_double))))
    return losses, grad_out


def _vol_args(volume, ctx):
    if len(volume.shape) != 3:
        raise ContractError("volume: expected a [nz, ny, nx] array")
    dev = _is_torch(volume) and volume.is_cuda
    if ctx is None:
        ctx = context(volume.device.index or 0) if dev else context(0)
    nz, ny, nx = (int(d) for d in volume.shape)
    return dev, ctx, (C.c_int * 3)(nx, ny, nz)


def volume_loss(rendered, target, alpha_ssim: float = 0.2, grad_out=None, ctx: Optional[Context] = None):
    """total_loss_fit (losses.hpp:648-664): L1 + alpha * SSIM3D on [nz, ny, nx] float32
    volumes. Returns ((l1, ssim, total), grad float32)."""
    if tuple(rendered.shape) != tuple(target.shape):
        raise ContractError("l1: volume shape mismatch")
    dev, ctx, dims = _vol_args(rendered, ctx)
    keep: list = []
    if grad_out is None:
        if dev:
            import torch
            grad_out = torch.empty(tuple(rendered.shape), dtype=torch.float32, device=rendered.device)
        else:
            grad_out = np.empty(tuple(rendered.shape), dtype=np.float32)
    rp, rl = _ptr(rendered if dev else np.ascontiguousarray(rendered, dtype=np.float32), keep)
    tp, tl = _ptr(target if dev else np.ascontiguousarray(target, dtype=np.float32), keep)
    gp, gl = _ptr(grad_out, keep)
    if not (rl == tl == gl):
        raise ContractError("volume_loss: rendered, target and grad must share one location")
    out = (C.c_double * 3)()
    ctx.check(ctx._lib.gsct_volume_loss(ctx.handle, C.c_void_p(rp), C.c_void_p(tp), dims, float(alpha_ssim),
                                        C.c_void_p(gp), rl, out))
    return (out[0], out[1], out[2]), grad_out


def tv3d(volume, grad_out=None, ctx: Optional[Context] = None):
    """tv3d (losses.hpp:530-595) on a [nz, ny, nx] float32 volume: (value, grad)."""
    dev, ctx, dims = _vol_args(volume, ctx)
    keep: list = []
    if grad_out is None:
        if dev:
            import torch
            grad_out = torch.empty(tuple(volume.shape), dtype=torch.float32, device=volume.device)
        else:
            grad_out = np.empty(tuple(volume.shape), dtype=np.float32)
    vp, vl = _ptr(volume if dev else np.ascontiguousarray(volume, dtype=np.float32), keep)
    gp, gl = _ptr(grad_out, keep)
    if vl != gl:
        raise ContractError("tv3d: volume and grad must share one location")
    val = C.c_double(0.0)
    ctx.check(ctx._lib.gsct_tv3d(ctx.handle, C.c_void_p(vp), dims, C.c_void_p(gp), vl, C.byref(val)))
    return float(val.value), grad_out


def raymarch_project(volume, grid: GridSpec, geometry: ScanGeometry, view_indices=None, out=None,
                     ctx: Optional[Context] = None):
    """raymarch_project (synthetic.hpp:171-232) of a [nz, ny, nx] float32 volume laid out on
    `grid` (origin = centre of voxel 0): images [V, n_v, n_u] float32, same kind as `volume`."""
    dev, ctx, _ = _vol_args(volume, ctx)
    if tuple(volume.shape) != (grid.dims[2], grid.dims[1], grid.dims[0]):
        raise ContractError("raymarch_project: volume shape does not match the grid")
    ang = _angles(geometry, view_indices)
    keep: list = []
    if out is None:
        if dev:
            import torch
            out = torch.empty((ang.size, geometry.n_v, geometry.n_u), dtype=torch.float32, device=volume.device)
        else:
            out = np.empty((ang.size, geometry.n_v, geometry.n_u), dtype=np.float32)
    vp, vl = _ptr(volume if dev else np.ascontiguousarray(volume, dtype=np.float32), keep)
    op, ol = _ptr(out, keep)
    gr = _grid_c(GridRegion.covering(grid))
    g = geometry.c()
    ctx.check(ctx._lib.gsct_raymarch_project(ctx.handle, C.c_void_p(vp), C.byref(gr), vl, C.byref(g),
                                             ang.ctypes.data_as(C.POINTER(C.c_double)), int(ang.size),
                                             C.c_void_p(op), ol))
    return out


@dataclass
class LearningRates:
    """optim.hpp:63-68"""
    position: float = 1e-4
    log_scale: float = 5e-3
    rotation: float = 1e-3
    density: float = 1e-2


def lr_schedule(base: float, final_lr: float, step: int, horizon: int) -> float:
    """lr_schedule (optim.hpp:71-78): log-linear decay from base to final over [0, horizon],
    clamped at final (host scalar, the reference's std::pow)."""
    if not (base > 0.0 and final_lr > 0.0):
        raise ContractError("lr_schedule: rates must be positive")
    if step <= 0:
        return float(base)
    if horizon <= 0 or step >= horizon:
        return float(final_lr)
    return float(base * (final_lr / base) ** (float(step) / float(horizon)))


def scene_extent(cloud: GaussianCloud) -> float:
    """scene_extent (core.hpp:120-129): half the diagonal of the positions' bounding box."""
    if cloud.size() == 0:
        raise ContractError("scene_extent: empty model")
    p = cloud.positions.cpu().numpy() if _is_torch(cloud.positions) else np.asarray(cloud.positions)
    return float(0.5 * np.linalg.norm(p.max(axis=0) - p.min(axis=0)))


class AdamState:
    """OptimState's Adam moments (optim.hpp:84-114) as device fp64 tensors."""

    def __init__(self, n: int, device: int = 0):
        import torch
        z = lambda *s: torch.zeros(s, dtype=torch.float64, device=f"cuda:{device}")
        self.m_pos, self.v_pos, self.m_ls, self.v_ls = z(n, 3), z(n, 3), z(n, 3), z(n, 3)
        self.m_rot, self.v_rot, self.m_dens, self.v_dens = z(n, 4), z(n, 4), z(n), z(n)
        self.step = 0
        self.skipped_updates = 0

    def _c(self) -> c_adam_state:
        arrs = (self.m_pos, self.v_pos, self.m_ls, self.v_ls, self.m_rot, self.v_rot, self.m_dens, self.v_dens)
        return c_adam_state(*[a.data_ptr() for a in arrs], self.step, self.skipped_updates)


def adam_step(cloud: GaussianCloud, state: AdamState, grads: ParamGradients, lrs: LearningRates = LearningRates(),
              ctx: Optional[Context] = None) -> None:
    """adam_step (optim.hpp:158-182) on a device-resident cloud (updated in place)."""
    if not cloud.on_device or not _is_torch(grads.positions):
        raise ContractError("adam_step: parameters and gradients must be device-resident")
    ctx = _ctx_for(cloud, ctx)
    keep: list = []
    cc = cloud._c(keep)
    st = state._c()
    gg = grads._c()
    lr = c_learning_rates(lrs.position, lrs.log_scale, lrs.rotation, lrs.density)
    ctx.check(ctx._lib.gsct_adam_step(ctx.handle, C.byref(cc), C.byref(st), C.byref(gg), C.byref(lr)))
    state.step = int(st.step)
    state.skipped_updates = int(st.skipped_updates)


# ---------------------------------------------------------------------------------------
# Adaptive density control
# ---------------------------------------------------------------------------------------
@dataclass
class ControlConfig:
    """TrainConfig's adaptive-control fields (optim.hpp:38-41)."""
    grad_threshold: float = 5e-5
    prune_density: float = 5e-4
    split_scale_fraction: float = 0.01
    max_gaussians: int = 100000


@dataclass
class AdaptiveReport:
    """optim.hpp:188-192"""
    pruned: int = 0
    cloned: int = 0
    split: int = 0


class OptimState(AdamState):
    """OptimState (optim.hpp:84-125) on device: the Adam moments plus the densification
    accumulators, all tracking the cloud size through adaptive control; the host Rng,
    scene extent and normalisation factor."""

    def __init__(self, n: int, seed: int = 0, device: int = 0):
        import torch
        super().__init__(n, device)
        self.accum_grad_norm = torch.zeros(n, dtype=torch.float64, device=f"cuda:{device}")
        self.accum_grad_dir = torch.zeros((n, 3), dtype=torch.float64, device=f"cuda:{device}")
        self.accum_count = torch.zeros(n, dtype=torch.int64, device=f"cuda:{device}")
        self.rng = Rng(seed)
        self.scene_extent = 1.0
        self.norm_factor = 1.0

    def check_lockstep(self, n: int) -> None:
        arrs = (self.m_pos, self.v_pos, self.m_ls, self.v_ls, self.m_rot, self.v_rot, self.m_dens, self.v_dens,
                self.accum_grad_norm, self.accum_grad_dir, self.accum_count)
        if any(a.shape[0] != n for a in arrs):
            raise ContractError("OptimState: arrays out of lockstep with the cloud")

    def _acc(self) -> c_control_accum:
        return c_control_accum(self.accum_grad_norm.data_ptr(), self.accum_grad_dir.data_ptr(),
                               self.accum_count.data_ptr())


def accumulate_control_stats(state: OptimState, grads: ParamGradients, ctx: Optional[Context] = None) -> None:
    """detail::accumulate_control_stats (optim.hpp:366-373) on device."""
    if not _is_torch(grads.positions):
        raise ContractError("accumulate_control_stats: gradients must be device-resident")
    n = int(grads.positions.shape[0])
    state.check_lockstep(n)
    ctx = ctx or context(grads.positions.device.index or 0)
    gg = grads._c()
    acc = state._acc()
    ctx.check(ctx._lib.gsct_accumulate_control_stats(ctx.handle, n, C.byref(gg), C.byref(acc)))


def adaptive_control(cloud: GaussianCloud, state: OptimState, config: ControlConfig = ControlConfig(),
                     ctx: Optional[Context] = None) -> AdaptiveReport:
    """adaptive_control (optim.hpp:201-317) on a device-resident cloud: prunes, clones and
    splits in place of `cloud` / `state` (their arrays are replaced) and returns the report.
    The split children draw from state.rng, whose engine state is left unchanged -- as in the
    reference, where the state is replaced by a copy taken before the draws (optim.hpp:244,
    301, 315)."""
    import torch
    if not cloud.on_device:
        raise ContractError("adaptive_control: clouds must be device-resident")
    n = cloud.size()
    state.check_lockstep(n)
    ctx = _ctx_for(cloud, ctx)
    dev = cloud.positions.device
    cap = max(n, int(config.max_gaussians))
    f64 = lambda *s: torch.empty(s, dtype=torch.float64, device=dev)
    out = GaussianCloud(f64(cap, 3), f64(cap, 3), f64(cap, 4), f64(cap))
    nxt = OptimState.__new__(OptimState)
    nxt.m_pos, nxt.v_pos, nxt.m_ls, nxt.v_ls = f64(cap, 3), f64(cap, 3), f64(cap, 3), f64(cap, 3)
    nxt.m_rot, nxt.v_rot, nxt.m_dens, nxt.v_dens = f64(cap, 4), f64(cap, 4), f64(cap), f64(cap)
    nxt.accum_grad_norm, nxt.accum_grad_dir = f64(cap), f64(cap, 3)
    nxt.accum_count = torch.empty(cap, dtype=torch.int64, device=dev)
    keep: list = []
    ci = cloud._c(keep)
    co = c_cloud(cap, out.positions.data_ptr(), out.log_scales.data_ptr(), out.rotations.data_ptr(),
                 out.raw_densities.data_ptr(), GSCT_DEVICE)
    si = state._c()
    nxt.step, nxt.skipped_updates = state.step, state.skipped_updates
    so = c_adam_state(*[a.data_ptr() for a in (nxt.m_pos, nxt.v_pos, nxt.m_ls, nxt.v_ls, nxt.m_rot, nxt.v_rot,
                                               nxt.m_dens, nxt.v_dens)], nxt.step, nxt.skipped_updates)
    rs = state.rng.state()
    cfg = c_control_config(config.grad_threshold, config.prune_density, config.split_scale_fraction,
                           state.scene_extent, int(config.max_gaussians))
    rep = c_adaptive_report()
    acc_in, acc_out = state._acc(), nxt._acc()
    ctx.check(ctx._lib.gsct_adaptive_control(ctx.handle, C.byref(ci), C.byref(si), C.byref(acc_in), C.byref(rs),
                                             C.byref(cfg), cap, C.byref(co), C.byref(so), C.byref(acc_out),
                                             C.byref(rep)))
    m = int(rep.n_next)
    cloud.positions, cloud.log_scales = out.positions[:m], out.log_scales[:m]
    cloud.rotations, cloud.raw_densities = out.rotations[:m], out.raw_densities[:m]
    for k in ("m_pos", "v_pos", "m_ls", "v_ls", "m_rot", "v_rot", "m_dens", "v_dens", "accum_grad_norm",
              "accum_grad_dir", "accum_count"):
        setattr(state, k, getattr(nxt, k)[:m])
    return AdaptiveReport(int(rep.pruned), int(rep.cloned), int(rep.split))


# ---------------------------------------------------------------------------------------
# Compressed model codec (FGSC, 22 bytes per splat)
# ---------------------------------------------------------------------------------------
def compress_model(cloud: GaussianCloud, ctx: Optional[Context] = None):
    """compress_model (io.hpp:323-385): (bytes, saturated). Host cloud -> numpy uint8 bytes;
    device cloud -> torch uint8 CUDA tensor (16 + 22 N)."""
    ctx = _ctx_for(cloud, ctx)
    keep: list = []
    cc = cloud._c(keep)
    n = cloud.size()
    sat = C.c_int64(0)
    if cloud.on_device:
        import torch
        out = torch.empty(16 + 22 * n, dtype=torch.uint8, device=cloud.positions.device)
        ctx.check(ctx._lib.gsct_compress_model(ctx.handle, C.byref(cc), C.c_void_p(out.data_ptr()), GSCT_DEVICE,
                                               C.byref(sat)))
    else:
        out = np.empty(16 + 22 * n, dtype=np.uint8)
        ctx.check(ctx._lib.gsct_compress_model(ctx.handle, C.byref(cc), C.c_void_p(out.ctypes.data), GSCT_HOST,
                                               C.byref(sat)))
    return out, int(sat.value)


def decompress_model(data, ctx: Optional[Context] = None) -> GaussianCloud:
    """decompress_model (io.hpp:387-419). numpy bytes -> host cloud; a torch uint8 CUDA
    tensor -> device cloud. Header errors raise ParseError with the reference's messages."""
    ctx = ctx or context(0)
    if _is_torch(data):
        import torch
        nb = int(data.numel())
        head = data[:16].cpu().numpy() if nb else np.zeros(0, dtype=np.uint8)
        ptr, loc, dev = data.data_ptr(), GSCT_DEVICE, data.device
    else:
        data = np.ascontiguousarray(data, dtype=np.uint8)
        nb = int(data.size)
        head = data[:16]
        ptr, loc, dev = (data.ctypes.data if nb else None), GSCT_HOST, None
    count = int.from_bytes(bytes(head[8:16]), "little") if len(head) >= 16 else 0
    n = count if nb == 16 + 22 * count else 0  # a size mismatch is reported by the call
    if dev is not None:
        import torch
        f = lambda *s: torch.empty(s, dtype=torch.float64, device=dev)
        cloud = GaussianCloud(f(n, 3), f(n, 3), f(n, 4), f(n))
        arrs = [cloud.positions, cloud.log_scales, cloud.rotations, cloud.raw_densities]
        co = c_cloud(count, *[a.data_ptr() for a in arrs], GSCT_DEVICE)
    else:
        cloud = GaussianCloud(np.empty((n, 3)), np.empty((n, 3)), np.empty((n, 4)), np.empty(n))
        arrs = [cloud.positions, cloud.log_scales, cloud.rotations, cloud.raw_densities]
        co = c_cloud(count, *[a.ctypes.data if a.size else None for a in arrs], GSCT_HOST)
    ctx.check(ctx._lib.gsct_decompress_model(ctx.handle, C.c_void_p(ptr) if ptr else None, nb, loc, C.byref(co)))
    return cloud
