"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the CPU checkers.

* `Orc`  — the plain-C restatement of the reference hot path (oracle/gsct_oracle.c,
           built into oracle/_build/liborc.so). Always available once built.
* `Ref`  — the UNCHANGED reference (/root/reference/proj/include/gsct/*.hpp) compiled with
           the test-only Eigen/Catch2 shims into oracle/_ref/libgsct_ref.so (built here,
           travels prebuilt to the GPU box). Also the CPU baseline of bench.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may
import this module. Inputs are duck-typed on the product's value types
(ScanGeometry / RasterSettings / VoxelSettings / GridRegion / GaussianCloud); every
array is float64 (images u fastest, volumes x fastest).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORC_LIB = HERE / "_build" / "liborc.so"
REF_LIB = HERE / "_ref" / "libgsct_ref.so"


class OracleError(RuntimeError):
    pass


class _Geo(C.Structure):
    _fields_ = [("cone", C.c_int), ("n_u", C.c_int), ("n_v", C.c_int), ("s_u", C.c_double), ("s_v", C.c_double),
                ("source_to_origin", C.c_double), ("origin_to_detector", C.c_double)]


class _RS(C.Structure):
    _fields_ = [("tau_cut", C.c_double), ("sigma_cap", C.c_double), ("dilation_px2", C.c_double),
                ("tile_size", C.c_int), ("dilate", C.c_int), ("bounding", C.c_int)]


class _VS(C.Structure):
    _fields_ = [("tau_cut", C.c_double), ("sigma_cap", C.c_double)]


class _Region(C.Structure):
    _fields_ = [("dims", C.c_int * 3), ("spacing", C.c_double), ("origin", C.c_double * 3)]


class _Stats(C.Structure):
    _fields_ = [("culled", C.c_int64), ("degenerate", C.c_int64), ("tile_pairs", C.c_int64),
                ("pixel_pairs", C.c_int64)]


class _Splat(C.Structure):
    _fields_ = [("mean2d", C.c_double * 2), ("cov2d", C.c_double * 4), ("conic", C.c_double * 4),
                ("amplitude", C.c_double), ("u_min", C.c_int), ("u_max", C.c_int), ("v_min", C.c_int),
                ("v_max", C.c_int), ("culled", C.c_int), ("degenerate", C.c_int)]


def _geo(g) -> _Geo:
    return _Geo(1 if g.mode == "cone" else 0, int(g.n_u), int(g.n_v), float(g.s_u), float(g.s_v),
                float(g.source_to_origin), float(g.origin_to_detector))


def _rs(r) -> _RS:
    return _RS(float(r.tau_cut), float(r.sigma_cap), float(r.dilation_px2), int(r.tile_size),
               1 if r.dilate else 0, 1 if r.bounding == "square_circumscribed" else 0)


def _vs(v) -> _VS:
    return _VS(float(v.tau_cut), float(v.sigma_cap))


def _region(r) -> _Region:
    return _Region((C.c_int * 3)(*[int(d) for d in r.dims]), float(r.spacing),
                   (C.c_double * 3)(*[float(o) for o in r.origin]))


def _cloud_arrays(cloud):
    f = lambda a: np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return f(cloud.positions), f(cloud.log_scales), f(cloud.rotations), f(cloud.raw_densities)


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a.size else None


def _grads(n: int):
    return dict(positions=np.zeros((n, 3)), log_scales=np.zeros((n, 3)), rotations=np.zeros((n, 4)),
                raw_densities=np.zeros(n), pos_grad_norm=np.zeros(n), visible=np.zeros(n, dtype=np.uint8))


def _gptrs(g):
    return [_p(g[k]) for k in ("positions", "log_scales", "rotations", "raw_densities", "pos_grad_norm", "visible")]


class Orc:
    """The C restatement (oracle/gsct_oracle.c)."""

    def __init__(self):
        if not ORC_LIB.exists():
            raise OracleError(f"{ORC_LIB} missing: run `make -C oracle oracle`")
        self.l = C.CDLL(str(ORC_LIB))
        self.l.orc_last_error.restype = C.c_char_p
        self.l.orc_max_eigenvalue_3x3.restype = C.c_double
        self.l.orc_bin_tiles.restype = C.c_int64

    def _chk(self, st):
        if st != 0:
            raise OracleError(self.l.orc_last_error().decode())

    def splat_bbox(self, g_peak, cov2d, mean2d, tau, n_u, n_v, sigma_cap=3.0, square=False):
        """projector.hpp:101-117 -> (visible, [u_min, u_max, v_min, v_max])."""
        cov = np.ascontiguousarray(cov2d, dtype=np.float64).reshape(4)
        mean = np.ascontiguousarray(mean2d, dtype=np.float64)
        rect = np.zeros(4, dtype=np.int32)
        ok = self.l.orc_splat_bbox(C.c_double(g_peak), _p(cov), _p(mean), C.c_double(tau), int(n_u), int(n_v),
                                   _p(rect), C.c_double(sigma_cap), 1 if square else 0)
        return bool(ok), rect.tolist()

    def rasterize_view(self, cloud, geom, view: int, rs):
        p, l, q, r = _cloud_arrays(cloud)
        img = np.zeros((geom.n_v, geom.n_u))
        st = _Stats()
        self._chk(self.l.orc_rasterize_view(C.c_int64(len(r)), _p(p), _p(l), _p(q), _p(r), C.byref(_geo(geom)),
                                            C.c_double(float(geom.angles[view])), C.byref(_rs(rs)), _p(img),
                                            C.byref(st)))
        return img, dict(culled=st.culled, degenerate=st.degenerate, tile_pairs=st.tile_pairs,
                         pixel_pairs=st.pixel_pairs)

    def rasterize_backward(self, cloud, geom, view: int, grad_image, rs):
        p, l, q, r = _cloud_arrays(cloud)
        gi = np.ascontiguousarray(grad_image, dtype=np.float64)
        g = _grads(len(r))
        self._chk(self.l.orc_rasterize_backward(C.c_int64(len(r)), _p(p), _p(l), _p(q), _p(r), C.byref(_geo(geom)),
                                                C.c_double(float(geom.angles[view])), _p(gi), C.byref(_rs(rs)),
                                                *_gptrs(g)))
        return g

    def project_cloud(self, cloud, geom, view: int, rs):
        p, l, q, r = _cloud_arrays(cloud)
        n = len(r)
        arr = (_Splat * max(n, 1))()
        self._chk(self.l.orc_project_cloud(C.c_int64(n), _p(p), _p(l), _p(q), _p(r), C.byref(_geo(geom)),
                                           C.c_double(float(geom.angles[view])), C.byref(_rs(rs)), arr))
        rect = np.array([[s.u_min, s.u_max, s.v_min, s.v_max] for s in arr[:n]], dtype=np.int32).reshape(n, 4)
        return dict(rect=rect, culled=np.array([bool(s.culled) for s in arr[:n]], dtype=bool),
                    degenerate=np.array([bool(s.degenerate) for s in arr[:n]], dtype=bool),
                    mean2d=np.array([list(s.mean2d) for s in arr[:n]]).reshape(n, 2),
                    conic=np.array([list(s.conic) for s in arr[:n]]).reshape(n, 4),
                    amplitude=np.array([s.amplitude for s in arr[:n]]), _raw=arr)

    def bin_tiles(self, cloud, geom, view: int, rs):
        """CSR (offsets[n_tiles+1], splats[pairs])."""
        pc = self.project_cloud(cloud, geom, view, rs)
        n = len(pc["amplitude"])
        ts = rs.tile_size
        n_tiles = ((geom.n_u + ts - 1) // ts) * ((geom.n_v + ts - 1) // ts)
        off = np.zeros(n_tiles + 1, dtype=np.int64)
        pairs = self.l.orc_bin_tiles(C.c_int64(n), pc["_raw"], int(geom.n_u), int(geom.n_v), int(ts), _p(off), None)
        vals = np.zeros(max(pairs, 1), dtype=np.int32)
        self.l.orc_bin_tiles(C.c_int64(n), pc["_raw"], int(geom.n_u), int(geom.n_v), int(ts), _p(off), _p(vals))
        return off, vals[:pairs]

    def voxelize(self, cloud, region, vs):
        p, l, q, r = _cloud_arrays(cloud)
        vol = np.zeros((region.dims[2], region.dims[1], region.dims[0]))
        st = _Stats()
        self._chk(self.l.orc_voxelize(C.c_int64(len(r)), _p(p), _p(l), _p(q), _p(r), C.byref(_region(region)),
                                      C.byref(_vs(vs)), _p(vol), C.byref(st)))
        return vol, dict(culled=st.culled, pixel_pairs=st.pixel_pairs)

    def voxelize_backward(self, cloud, region, grad_volume, vs):
        p, l, q, r = _cloud_arrays(cloud)
        gv = np.ascontiguousarray(grad_volume, dtype=np.float64)
        g = _grads(len(r))
        self._chk(self.l.orc_voxelize_backward(C.c_int64(len(r)), _p(p), _p(l), _p(q), _p(r),
                                               C.byref(_region(region)), _p(gv), C.byref(_vs(vs)), *_gptrs(g)))
        return g

    def prepare_voxel_splats(self, cloud, region, vs):
        p, l, q, r = _cloud_arrays(cloud)
        n = len(r)
        lo = np.zeros((n, 3), dtype=np.int32)
        hi = np.zeros((n, 3), dtype=np.int32)
        skip = np.zeros(n, dtype=np.uint8)
        self._chk(self.l.orc_prepare_voxel_splats(C.c_int64(n), _p(p), _p(l), _p(q), _p(r), C.byref(_region(region)),
                                                  C.byref(_vs(vs)), _p(lo), _p(hi), _p(skip), None))
        return lo, hi, skip.astype(bool)


class Ref:
    """The unchanged reference compiled here (oracle/_ref/libgsct_ref.so)."""

    def __init__(self, threads: int | None = None):
        if not REF_LIB.exists():
            raise OracleError(f"{REF_LIB} missing: run `make -C oracle ref` where /root/reference exists")
        self.l = C.CDLL(str(REF_LIB))
        self.l.ref_last_error.restype = C.c_char_p
        self.l.ref_cloud_create.restype = C.c_void_p
        self.l.ref_cloud_create.argtypes = [C.c_int64] + [C.c_void_p] * 4
        self.l.ref_cloud_destroy.argtypes = [C.c_void_p]
        self.l.ref_synthetic_cloud.restype = C.c_int64
        self.l.ref_synthetic_cloud.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double,
                                               C.c_uint64] + [C.c_void_p] * 4
        if threads is not None:
            self.l.ref_set_threads(int(threads))

    def threads(self) -> int:
        return int(self.l.ref_thread_count())

    def set_threads(self, n: int) -> None:
        self.l.ref_set_threads(int(n))

    def _chk(self, st):
        if st != 0:
            raise OracleError(self.l.ref_last_error().decode())

    def cloud(self, cloud):
        """Opaque reference GaussianCloud (freed with free_cloud)."""
        p, l, q, r = _cloud_arrays(cloud)
        return self.l.ref_cloud_create(C.c_int64(len(r)), _p(p), _p(l), _p(q), _p(r))

    def free_cloud(self, h) -> None:
        self.l.ref_cloud_destroy(h)

    def _angles(self, geom):
        return np.ascontiguousarray(np.asarray(geom.angles, dtype=np.float64))

    def rasterize_view(self, h, geom, view: int, rs):
        ang = self._angles(geom)
        img = np.zeros((geom.n_v, geom.n_u))
        st = _Stats()
        ms = np.zeros(2)
        self._chk(self.l.ref_rasterize_view(C.c_void_p(h), C.byref(_geo(geom)), _p(ang), len(ang), int(view),
                                            C.byref(_rs(rs)), _p(img), C.byref(st), _p(ms)))
        return img, dict(culled=st.culled, degenerate=st.degenerate, tile_pairs=st.tile_pairs,
                         pixel_pairs=st.pixel_pairs, forward_ms=ms[0])

    def rasterize_backward(self, h, geom, view: int, grad_image, rs, n: int):
        ang = self._angles(geom)
        gi = np.ascontiguousarray(grad_image, dtype=np.float64)
        g = _grads(n)
        ms = np.zeros(2)
        self._chk(self.l.ref_rasterize_backward(C.c_void_p(h), C.byref(_geo(geom)), _p(ang), len(ang), int(view),
                                                _p(gi), C.byref(_rs(rs)), *_gptrs(g), _p(ms)))
        g["backward_ms"] = ms[1]
        return g

    def project_and_bin(self, h, geom, view: int, rs, n: int):
        ang = self._angles(geom)
        ts = rs.tile_size
        n_tiles = ((geom.n_u + ts - 1) // ts) * ((geom.n_v + ts - 1) // ts)
        rect = np.zeros((n, 4), dtype=np.int32)
        culled = np.zeros(n, dtype=np.uint8)
        degen = np.zeros(n, dtype=np.uint8)
        mean2d = np.zeros((n, 2))
        conic = np.zeros((n, 4))
        amp = np.zeros(n)
        off = np.zeros(n_tiles + 1, dtype=np.int64)
        npairs = C.c_int64(0)
        args = [C.c_void_p(h), C.byref(_geo(geom)), _p(ang), len(ang), int(view), C.byref(_rs(rs)), _p(rect),
                _p(culled), _p(degen), _p(mean2d), _p(conic), _p(amp)]
        self._chk(self.l.ref_project_and_bin(*args, None, None, C.byref(npairs)))
        vals = np.zeros(max(npairs.value, 1), dtype=np.int32)
        self._chk(self.l.ref_project_and_bin(*args, _p(off), _p(vals), C.byref(npairs)))
        return dict(rect=rect, culled=culled.astype(bool), degenerate=degen.astype(bool), mean2d=mean2d,
                    conic=conic, amplitude=amp, tile_offsets=off, tile_splats=vals[: npairs.value])

    def voxelize(self, h, region, vs):
        vol = np.zeros((region.dims[2], region.dims[1], region.dims[0]))
        st = _Stats()
        ms = np.zeros(2)
        self._chk(self.l.ref_voxelize(C.c_void_p(h), C.byref(_region(region)), C.byref(_vs(vs)), _p(vol),
                                      C.byref(st), _p(ms)))
        return vol, dict(culled=st.culled, pixel_pairs=st.pixel_pairs, forward_ms=ms[0])

    def voxelize_backward(self, h, region, grad_volume, vs, n: int):
        gv = np.ascontiguousarray(grad_volume, dtype=np.float64)
        g = _grads(n)
        ms = np.zeros(2)
        self._chk(self.l.ref_voxelize_backward(C.c_void_p(h), C.byref(_region(region)), _p(gv), C.byref(_vs(vs)),
                                               *_gptrs(g), _p(ms)))
        g["backward_ms"] = ms[1]
        return g

    def prepare_voxel_splats(self, h, region, vs, n: int):
        lo = np.zeros((n, 3), dtype=np.int32)
        hi = np.zeros((n, 3), dtype=np.int32)
        skip = np.zeros(n, dtype=np.uint8)
        self._chk(self.l.ref_prepare_voxel_splats(C.c_void_p(h), C.byref(_region(region)), C.byref(_vs(vs)), _p(lo),
                                                  _p(hi), _p(skip)))
        return lo, hi, skip.astype(bool)

    def synthetic_cloud(self, count, half_extent=0.8, scale=0.04, anisotropy=1.0, density=1.0, seed=0):
        pos = np.zeros((count, 3))
        ls = np.zeros((count, 3))
        q = np.zeros((count, 4))
        raw = np.zeros(count)
        self.l.ref_synthetic_cloud(count, half_extent, scale, anisotropy, density, seed, _p(pos), _p(ls), _p(q),
                                   _p(raw))
        return pos, ls, q, raw

    def shepp_logan_cloud(self, count: int, side: int, spacing: float = 1.0, seed: int = 0):
        """The benchmark phantom cloud drawn with the reference's Rng (ref_shepp_logan_cloud)."""
        pos = np.zeros((count, 3))
        ls = np.zeros((count, 3))
        q = np.zeros((count, 4))
        raw = np.zeros(count)
        self.l.ref_shepp_logan_cloud(C.c_int64(count), C.c_double(side), C.c_double(spacing), C.c_uint64(seed),
                                     _p(pos), _p(ls), _p(q), _p(raw))
        return pos, ls, q, raw

    def default_geometry(self, dims, spacing, n_views, cone, n_u, n_v):
        g = _Geo()
        ang = np.zeros(n_views)
        self.l.ref_default_geometry(int(dims[0]), int(dims[1]), int(dims[2]), C.c_double(spacing), int(n_views),
                                    int(cone), int(n_u), int(n_v), C.byref(g), _p(ang))
        return g, ang

    # -- next-row operators (unchanged reference losses.hpp / optim.hpp) --------------
    def total_loss_recon(self, rendered: np.ndarray, measured: np.ndarray, alpha_ssim: float):
        """(l1, ssim, total), grad for one image (losses.hpp:613-637, alpha_tv = 0)."""
        r = np.ascontiguousarray(rendered, dtype=np.float64)
        m = np.ascontiguousarray(measured, dtype=np.float64)
        g = np.zeros_like(r)
        out = np.zeros(3)
        f = self.l.ref_total_loss_recon
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_void_p]
        self._chk(f(_p(r), _p(m), r.shape[1], r.shape[0], float(alpha_ssim), _p(g), _p(out)))
        return out, g

    def adam_step(self, params: dict, moments: dict, grads: dict, lrs, step: int, skipped: int):
        """adam_step (optim.hpp:158-182) on flat fp64 arrays, updated in place; returns
        (step, skipped)."""
        f = self.l.ref_adam_step
        f.argtypes = [C.c_int64] + [C.c_void_p] * 4 + [C.c_void_p] + [C.c_void_p] * 4 + [C.c_void_p] * 3
        keys = ("m_pos", "v_pos", "m_ls", "v_ls", "m_rot", "v_rot", "m_dens", "v_dens")
        mv = (C.c_void_p * 8)(*[moments[k].ctypes.data for k in keys])
        lr = np.array([lrs.position, lrs.log_scale, lrs.rotation, lrs.density], dtype=np.float64)
        st = C.c_int64(step)
        sk = C.c_int64(skipped)
        n = len(params["raw"])
        self._chk(f(n, _p(params["pos"]), _p(params["ls"]), _p(params["q"]), _p(params["raw"]), mv, _p(grads["pos"]),
                    _p(grads["ls"]), _p(grads["q"]), _p(grads["raw"]), _p(lr), C.byref(st), C.byref(sk)))
        return int(st.value), int(sk.value)


    def adaptive_control(self, params: dict, moments: dict, acc: dict, rng_state: np.ndarray, grad_threshold: float,
                         prune_density: float, split_scale_fraction: float, scene_extent: float,
                         max_gaussians: int):
        """adaptive_control (optim.hpp:201-317) of the unchanged reference on flat fp64 arrays.
        rng_state: uint64[313] = the engine's x[0..311], p (advanced in place). Returns
        (params, moments, report {pruned, cloned, split, n_next}) of the output cloud."""
        n = len(params["raw"])
        cap = max(n, int(max_gaussians))
        f = self.l.ref_adaptive_control
        f.argtypes = [C.c_int64] + [C.c_void_p] * 4 + [C.c_void_p] * 4 + [C.c_void_p] * 2 + [C.c_int64, C.c_int64] + \
                     [C.c_void_p] * 4 + [C.c_void_p, C.c_void_p]
        keys = ("m_pos", "v_pos", "m_ls", "v_ls", "m_rot", "v_rot", "m_dens", "v_dens")
        width = {"m_pos": 3, "v_pos": 3, "m_ls": 3, "v_ls": 3, "m_rot": 4, "v_rot": 4, "m_dens": 1, "v_dens": 1}
        mv_in = [np.ascontiguousarray(moments[k], dtype=np.float64) for k in keys]
        mv = (C.c_void_p * 8)(*[a.ctypes.data for a in mv_in])
        out_m = {k: np.zeros((cap, width[k]) if width[k] > 1 else (cap,)) for k in keys}
        omv = (C.c_void_p * 8)(*[out_m[k].ctypes.data for k in keys])
        out_p = {"pos": np.zeros((cap, 3)), "ls": np.zeros((cap, 3)), "q": np.zeros((cap, 4)), "raw": np.zeros(cap)}
        cfg = np.array([grad_threshold, prune_density, split_scale_fraction, scene_extent], dtype=np.float64)
        rep = np.zeros(4, dtype=np.int64)
        assert rng_state.dtype == np.uint64 and rng_state.shape == (313,)
        ins = {k: np.ascontiguousarray(params[k], dtype=np.float64) for k in ("pos", "ls", "q", "raw")}
        an = np.ascontiguousarray(acc["grad_norm"], dtype=np.float64)
        ad = np.ascontiguousarray(acc["grad_dir"], dtype=np.float64)
        ac = np.ascontiguousarray(acc["count"], dtype=np.int64)
        self._chk(f(n, _p(ins["pos"]), _p(ins["ls"]), _p(ins["q"]), _p(ins["raw"]), mv, _p(an), _p(ad), ac.ctypes.data,
                    rng_state.ctypes.data, _p(cfg), int(max_gaussians), cap, _p(out_p["pos"]), _p(out_p["ls"]),
                    _p(out_p["q"]), _p(out_p["raw"]), omv, rep.ctypes.data))
        m = int(rep[3])
        return ({k: v[:m] for k, v in out_p.items()}, {k: v[:m] for k, v in out_m.items()},
                {"pruned": int(rep[0]), "cloned": int(rep[1]), "split": int(rep[2]), "n_next": m})

    def compress_model(self, params: dict):
        """compress_model (io.hpp:323-385): (bytes, saturated)."""
        n = len(params["raw"])
        out = np.zeros(16 + 22 * n, dtype=np.uint8)
        sat = C.c_int64(0)
        f = self.l.ref_compress_model
        f.argtypes = [C.c_int64] + [C.c_void_p] * 5 + [C.c_void_p]
        ins = {k: np.ascontiguousarray(params[k], dtype=np.float64) for k in ("pos", "ls", "q", "raw")}
        self._chk(f(n, _p(ins["pos"]), _p(ins["ls"]), _p(ins["q"]), _p(ins["raw"]), out.ctypes.data, C.byref(sat)))
        return out, int(sat.value)

    def decompress_model(self, data: np.ndarray, capacity: int = 1 << 16):
        """decompress_model (io.hpp:387-419): dict of pos / ls / q / raw."""
        data = np.ascontiguousarray(data, dtype=np.uint8)
        cap = max(int(capacity), 1)
        out = {"pos": np.zeros((cap, 3)), "ls": np.zeros((cap, 3)), "q": np.zeros((cap, 4)), "raw": np.zeros(cap)}
        m = C.c_int64(0)
        f = self.l.ref_decompress_model
        f.argtypes = [C.c_void_p, C.c_int64, C.c_int64] + [C.c_void_p] * 4 + [C.c_void_p]
        self._chk(f(data.ctypes.data if data.size else None, data.size, cap, _p(out["pos"]), _p(out["ls"]),
                    _p(out["q"]), _p(out["raw"]), C.byref(m)))
        return {k: v[:m.value] for k, v in out.items()}

    def total_loss_fit(self, rendered: np.ndarray, target: np.ndarray, alpha_ssim: float, streaming: bool = True):
        """(l1, ssim, total), grad for a [nz, ny, nx] volume (losses.hpp:648-664)."""
        r = np.ascontiguousarray(rendered, dtype=np.float64)
        t = np.ascontiguousarray(target, dtype=np.float64)
        dims = np.array([r.shape[2], r.shape[1], r.shape[0]], dtype=np.int32)
        g = np.zeros_like(r)
        out = np.zeros(3)
        f = self.l.ref_total_loss_fit
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_void_p, C.c_void_p]
        self._chk(f(_p(r), _p(t), dims.ctypes.data, float(alpha_ssim), 1 if streaming else 0, _p(g), _p(out)))
        return out, g

    def tv3d(self, volume: np.ndarray):
        """value, grad (losses.hpp:530-595) for a [nz, ny, nx] volume."""
        v = np.ascontiguousarray(volume, dtype=np.float64)
        dims = np.array([v.shape[2], v.shape[1], v.shape[0]], dtype=np.int32)
        g = np.zeros_like(v)
        val = C.c_double(0)
        f = self.l.ref_tv3d
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        self._chk(f(_p(v), dims.ctypes.data, _p(g), C.byref(val)))
        return float(val.value), g

    def raymarch_project(self, volume: np.ndarray, spacing: float, origin, geom):
        """raymarch_project (synthetic.hpp:171-232): images [n_angles, n_v, n_u]."""
        v = np.ascontiguousarray(volume, dtype=np.float64)
        dims = np.array([v.shape[2], v.shape[1], v.shape[0]], dtype=np.int32)
        org = np.ascontiguousarray(origin, dtype=np.float64)
        ang = self._angles(geom)
        out = np.zeros((len(ang), geom.n_v, geom.n_u))
        f = self.l.ref_raymarch_project
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        self._chk(f(_p(v), dims.ctypes.data, float(spacing), _p(org), C.byref(_geo(geom)), _p(ang), len(ang), _p(out)))
        return out

def _ref_random_cloud(self, seed, count, pos_range=5.0, scale_lo=0.5, scale_hi=2.5):
    pos = np.zeros((count, 3))
    ls = np.zeros((count, 3))
    q = np.zeros((count, 4))
    raw = np.zeros(count)
    self.l.ref_random_cloud(C.c_uint64(seed), int(count), C.c_double(pos_range), C.c_double(scale_lo),
                            C.c_double(scale_hi), _p(pos), _p(ls), _p(q), _p(raw))
    return pos, ls, q, raw


Ref.random_cloud = _ref_random_cloud
