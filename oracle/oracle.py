"""ctypes front end of the C parity oracle (oracle/ges_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  Never by the product package
(paper_2402_10128_b200), which must fail loudly without its CUDA library.

Every function mirrors a stage of the paper's method:
  preprocess      S1   Eq. 2, 4, 6; PAPER.md:242-294 (ges_geom.inc)
  pairs_sorted    S2   brute-force keys (tile<<32 | depth bits) + sort
  tile_lists      S2/S3 per-tile membership lists, sorted by (depth, index)
  render_fwd      S4   Eq. 3 front-to-back compositing in fp64
  render_bwd      S5a  hand-derived adjoint of Eq. 3 in fp64
  backward_particles S5b chain rule to the raw parameters incl. beta
  render / render_and_grad  the full definitional pipeline.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libges_oracle.so")
_SRC = [os.path.join(_HERE, "ges_oracle.c"), os.path.join(_HERE, "ges_geom.inc")]
_lock = threading.Lock()
_lib = None

VISIBLE, CULL_NEAR, DEGENERATE, OFFSCREEN = 0, 1, 2, 3
PHI_SCALE, PHI_VARIANCE = 0, 1

GCC_FLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, contraction off).  Building the checker is not
    using it; __graft_entry__.build() calls this."""
    stale = force or not os.path.exists(_SO) or any(
        os.path.getmtime(s) > os.path.getmtime(_SO) for s in _SRC)
    if stale:
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *GCC_FLAGS, "-o", tmp, _SRC[0], "-lm"], cwd=_HERE)
        os.replace(tmp, _SO)
    return _SO


class _Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("near_z", C.c_float), ("R", C.c_float * 9),
                ("t", C.c_float * 3)]


class _Settings(C.Structure):
    _fields_ = [("rho", C.c_float), ("phi_mode", C.c_int32), ("gaussian_only", C.c_int32),
                ("bg", C.c_float * 3), ("kernel", C.c_int32)]


def _particles_struct(ctype):
    class _P(C.Structure):
        _fields_ = [("P", C.c_int64), ("sh_degree", C.c_int32)] + [
            (n, C.POINTER(ctype)) for n in ("mean", "log_scale", "quat", "opacity_logit", "sh", "beta")]
    return _P


def _pre_struct(ctype):
    class _Pre(C.Structure):
        _fields_ = [(n, C.POINTER(ctype)) for n in ("depth", "uv", "conic", "cov2d", "kappa", "rgb")] + [
            (n, C.POINTER(C.c_int32)) for n in ("radius", "rect", "rect3", "tiles", "status", "flags")]
    return _Pre


_PartF32, _PartF64 = _particles_struct(C.c_float), _particles_struct(C.c_double)
_PreF32, _PreF64 = _pre_struct(C.c_float), _pre_struct(C.c_double)


class _Screen(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32),
                ("bg", C.c_double * 3)]


class _Geom(C.Structure):
    _fields_ = [("precision", C.c_int32), ("_pad", C.c_int32), ("P", C.c_int64), ("uv", C.c_void_p),
                ("conic", C.c_void_p), ("kappa", C.c_void_p)]


class _Splat2D(C.Structure):
    _fields_ = [("P", C.c_int64)] + [(n, C.POINTER(C.c_double)) for n in ("uv", "conic", "kappa", "rgb", "hbeta")]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_SO)
            L.or_exp_spec.restype = C.c_float
            L.or_exp_spec.argtypes = [C.c_float]
            L.or_count_pairs.restype = C.c_int64
            L.or_pairs_sorted.restype = C.c_int64
            L.or_tile_lists.restype = C.c_int64
            L.or_num_threads.restype = C.c_int
            _lib = L
    return _lib


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def num_threads() -> int:
    return int(lib().or_num_threads())


def set_num_threads(n: int) -> None:
    lib().or_set_num_threads(C.c_int(int(n)))


# ---------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------
KERNEL_PHI_GAUSS, KERNEL_EXACT_BETA = 0, 1


@dataclass
class Settings:
    rho: float = 0.1
    phi_mode: int = PHI_SCALE
    gaussian_only: int = 0
    background: tuple = (0.0, 0.0, 0.0)
    kernel: int = KERNEL_PHI_GAUSS  # 1: the exact GEF kernel of Eq. 2


def _cam(cam) -> _Camera:
    c = _Camera()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy, c.near_z = cam.fx, cam.fy, cam.cx, cam.cy, cam.near
    R = np.asarray(cam.R, np.float32).reshape(9)
    t = np.asarray(cam.t, np.float32).reshape(3)
    for k in range(9):
        c.R[k] = float(R[k])
    for k in range(3):
        c.t[k] = float(t[k])
    return c


def _settings(st: Settings) -> _Settings:
    s = _Settings()
    s.rho, s.phi_mode, s.gaussian_only = st.rho, int(st.phi_mode), int(st.gaussian_only)
    s.kernel = int(st.kernel)
    for k in range(3):
        s.bg[k] = float(st.background[k])
    return s


class _Keep:
    """Holds numpy arrays alive while ctypes structs point into them."""

    def __init__(self):
        self.items = []

    def __call__(self, a):
        self.items.append(a)
        return a


def _part_struct(parts, dtype, keep):
    S = _PartF32 if dtype == np.float32 else _PartF64
    ct = C.c_float if dtype == np.float32 else C.c_double
    s = S()
    s.P = parts.P
    s.sh_degree = parts.sh_degree
    for n in ("mean", "log_scale", "quat", "opacity_logit", "sh", "beta"):
        a = keep(np.ascontiguousarray(getattr(parts, n), dtype=dtype))
        setattr(s, n, _ptr(a, ct))
    return s


# ---------------------------------------------------------------------------
# S1
# ---------------------------------------------------------------------------
def preprocess(parts, cam, st: Settings, precision: str = "f32") -> dict:
    """Per-particle stage S1.  precision 'f32' = KEYSPEC (bit-exact with the
    kernel), 'f64' = the same formulas in double."""
    dtype = np.float32 if precision == "f32" else np.float64
    ct = C.c_float if precision == "f32" else C.c_double
    P = parts.P
    keep = _Keep()
    ps = _part_struct(parts, dtype, keep)
    out = {
        "depth": np.zeros(P, dtype), "uv": np.zeros((2, P), dtype), "conic": np.zeros((3, P), dtype),
        "cov2d": np.zeros((3, P), dtype), "kappa": np.zeros(P, dtype), "rgb": np.zeros((3, P), dtype),
        "radius": np.zeros(P, np.int32), "rect": np.zeros((4, P), np.int32), "rect3": np.zeros((4, P), np.int32),
        "tiles": np.zeros(P, np.int32), "status": np.zeros(P, np.int32), "flags": np.zeros(P, np.int32),
    }
    pre = (_PreF32 if precision == "f32" else _PreF64)()
    for n in ("depth", "uv", "conic", "cov2d", "kappa", "rgb"):
        setattr(pre, n, _ptr(out[n], ct))
    for n in ("radius", "rect", "rect3", "tiles", "status", "flags"):
        setattr(pre, n, _ptr(out[n], C.c_int32))
    c, s = _cam(cam), _settings(st)
    fn = lib().or_preprocess_f32 if precision == "f32" else lib().or_preprocess_f64
    fn(C.byref(ps), C.byref(c), C.byref(s), C.byref(pre))
    out["precision"] = precision
    # exact GEF kernel: beta / 2 per particle for the compositing (exact halving of the stored beta)
    out["hbeta"] = 0.5 * np.asarray(parts.beta, dtype).astype(np.float64) if int(st.kernel) == 1 else None
    out["tiles_x"] = (cam.width + 15) // 16
    out["tiles_y"] = (cam.height + 15) // 16
    return out


def depth_order_key(pre) -> np.ndarray:
    """Depth as a monotone unsigned integer key (the fp32 bit pattern for the
    KEYSPEC path; the fp64 bit pattern otherwise).  Depth > near > 0."""
    d = pre["depth"]
    if d.dtype == np.float32:
        return d.view(np.uint32).astype(np.uint64)
    return d.view(np.uint64).copy()


# ---------------------------------------------------------------------------
# S2 / S3
# ---------------------------------------------------------------------------
def count_pairs(pre) -> int:
    return int(lib().or_count_pairs(C.c_int64(pre["status"].size), _ptr(pre["status"], C.c_int32),
                                    _ptr(pre["tiles"], C.c_int32)))


MEMBERSHIPS = ("rect", "exact", "all", "sigma3")


def _membership(pre, membership):
    """(status, rect, tile-test geometry or None) of a membership rule:
    'rect'   = the R10 rect (the tight alpha >= 0.98/255 box; the kernel's rule),
    'exact'  = R10 rect AND the tile itself reaches alpha >= 0.98/255 (R8 test),
    'all'    = every particle that passed the geometric tests, in every tile
               (the definitional sum of Eq. 3 with the alpha skip; brute force),
    'sigma3' = the inherited 3-sigma rect (R7; a different, truncating rule).
    'rect', 'exact' and 'all' give identical images and gradients (pinned in
    test_oracle_pins)."""
    assert membership in MEMBERSHIPS, membership
    st = pre["status"]
    if membership == "sigma3":
        return st, np.ascontiguousarray(pre["rect3"]), None
    if membership == "all":
        st = np.where(st == OFFSCREEN, VISIBLE, st).astype(np.int32)
        rect = np.zeros_like(pre["rect"])
        rect[2], rect[3] = pre["tiles_x"], pre["tiles_y"]
        return st, rect, None
    if membership == "rect":
        return st, pre["rect"], None
    g = _Geom()
    g.precision = 0 if pre["precision"] == "f32" else 1
    g.P = pre["status"].size
    g.uv, g.conic, g.kappa = pre["uv"].ctypes.data, pre["conic"].ctypes.data, pre["kappa"].ctypes.data
    return st, pre["rect"], g


def _rect_pairs(status, rect) -> int:
    vis = status == VISIBLE
    area = (rect[2] - rect[0]).astype(np.int64) * (rect[3] - rect[1]).astype(np.int64)
    return int(area[vis].sum())


def pairs_sorted(pre, membership="rect"):
    """All (key, particle) pairs sorted by (key, index); key = tile<<32 | depth bits."""
    assert pre["precision"] == "f32"
    P = pre["status"].size
    st, rect, g = _membership(pre, membership)
    M = _rect_pairs(st, rect)  # rect pairs: an upper bound
    keys = np.zeros(max(M, 1), np.uint64)
    vals = np.zeros(max(M, 1), np.int32)
    db = np.ascontiguousarray(pre["depth"].view(np.uint32))
    got = lib().or_pairs_sorted(C.c_int64(P), _ptr(st, C.c_int32), _ptr(rect, C.c_int32),
                                _ptr(db, C.c_uint32), C.byref(g) if g is not None else None,
                                C.c_int32(pre["tiles_x"]), _ptr(keys, C.c_uint64), _ptr(vals, C.c_int32),
                                C.c_int64(keys.size))
    assert 0 <= got <= M, (got, M)
    return keys[:got], vals[:got]


def tile_lists(pre, tile_mask: Optional[np.ndarray] = None, membership="rect"):
    """Per-tile membership lists sorted by (depth key, index): (offsets[T+1], list)."""
    P = pre["status"].size
    T = pre["tiles_x"] * pre["tiles_y"]
    order = np.ascontiguousarray(depth_order_key(pre))
    if membership == "all" and tile_mask is not None:
        # every geometrically valid particle in every selected tile: each selected tile's
        # list is the same (depth key, index) order of all of them (the definitional sum)
        st, _, _ = _membership(pre, membership)
        ids = np.nonzero(st == VISIBLE)[0]
        srt = ids[np.lexsort((ids, order[ids]))].astype(np.int32)
        sel = np.ascontiguousarray(tile_mask, dtype=np.uint8) != 0
        offsets = np.concatenate([[0], np.cumsum(sel.astype(np.int64) * srt.size)])
        return offsets, np.tile(srt, int(sel.sum()))
    offsets = np.zeros(T + 1, np.int64)
    mask_p = None
    if tile_mask is not None:
        tile_mask = np.ascontiguousarray(tile_mask, dtype=np.uint8)
        mask_p = _ptr(tile_mask, C.c_uint8)
    st, rect, g = _membership(pre, membership)
    args = (C.c_int64(P), _ptr(st, C.c_int32), _ptr(rect, C.c_int32), _ptr(order, C.c_uint64),
            C.byref(g) if g is not None else None, C.c_int32(pre["tiles_x"]), C.c_int32(pre["tiles_y"]), mask_p,
            _ptr(offsets, C.c_int64))
    total = lib().or_tile_lists(*args, None, C.c_int64(0))
    lst = np.zeros(max(total, 1), np.int32)
    got = lib().or_tile_lists(*args, _ptr(lst, C.c_int32), C.c_int64(lst.size))
    assert got == total
    return offsets, lst[:total]


# ---------------------------------------------------------------------------
# S4 / S5a / S5b
# ---------------------------------------------------------------------------
def _screen(cam, st):
    s = _Screen()
    s.width, s.height = cam.width, cam.height
    s.tiles_x, s.tiles_y = (cam.width + 15) // 16, (cam.height + 15) // 16
    for k in range(3):
        s.bg[k] = float(np.float32(st.background[k]))
    return s


def _splat(pre, keep):
    s = _Splat2D()
    s.P = pre["status"].size
    for n in ("uv", "conic", "kappa", "rgb"):
        a = keep(np.ascontiguousarray(pre[n], dtype=np.float64))
        setattr(s, n, _ptr(a, C.c_double))
    if pre.get("hbeta") is not None:
        s.hbeta = _ptr(keep(np.ascontiguousarray(pre["hbeta"], dtype=np.float64)), C.c_double)
    return s


def render_fwd(pre, cam, st: Settings, offsets, lst, tile_mask=None) -> dict:
    """Eq. 3 compositing in fp64 of the per-particle state `pre`."""
    H, W = cam.height, cam.width
    keep = _Keep()
    sp = _splat(pre, keep)
    img = np.zeros((3, H, W), np.float64)
    fT = np.zeros((H, W), np.float64)
    nc = np.zeros((H, W), np.int32)
    ne = np.zeros((H, W), np.int32)
    ncomp = np.zeros((H, W), np.int32)
    amb = np.zeros((H, W), np.uint8)
    mp = None
    if tile_mask is not None:
        tile_mask = keep(np.ascontiguousarray(tile_mask, dtype=np.uint8))
        mp = _ptr(tile_mask, C.c_uint8)
    lst = keep(np.ascontiguousarray(lst if lst.size else np.zeros(1, np.int32), dtype=np.int32))
    lib().or_render_fwd(C.byref(_screen(cam, st)), C.byref(sp), _ptr(offsets, C.c_int64), _ptr(lst, C.c_int32), mp,
                        _ptr(img, C.c_double), _ptr(fT, C.c_double), _ptr(nc, C.c_int32), _ptr(ne, C.c_int32),
                        _ptr(ncomp, C.c_int32), _ptr(amb, C.c_uint8))
    return {"image": img, "final_T": fT, "n_contrib": nc, "n_eval": ne, "n_comp": ncomp, "amb": amb}


def render_fwd_alternatives(pre, cam, st: Settings, offsets, lst, amb, n_alt: int = 4) -> np.ndarray:
    """R18, both branches: for every pixel the oracle flags (amb != 0),
    alt[f] = the image when the f-th threshold-ambiguous decision of the pixel (in
    list order: a 0.99 clamp, a 1/255 skip or a T < 1e-4 stop) takes its other
    outcome, every other decision as usual; NaN where the pixel has no f-th such
    decision.  An fp32 implementation may land on either side of any of them."""
    H, W = cam.height, cam.width
    keep = _Keep()
    sp = _splat(pre, keep)
    alt = np.zeros((n_alt, 3, H, W), np.float64)
    lst = keep(np.ascontiguousarray(lst if lst.size else np.zeros(1, np.int32), dtype=np.int32))
    amb = keep(np.ascontiguousarray(amb, dtype=np.uint8))
    lib().or_render_fwd_alternatives(C.byref(_screen(cam, st)), C.byref(sp), _ptr(offsets, C.c_int64),
                                     _ptr(lst, C.c_int32), _ptr(amb, C.c_uint8), C.c_int(int(n_alt)),
                                     _ptr(alt, C.c_double))
    return alt


def render_bwd(pre, cam, st: Settings, offsets, lst, dL_dimg, tile_mask=None, with_abs: bool = False):
    """S5a: per-particle 2D gradients g2d [10][P] = (du, dv, da, db, dc, dkappa, dr, dg, db, dbeta);
    dbeta (the exact GEF kernel's direct shape term) is 0 for the phi-bar Gaussian kernel.
    with_abs: also return the R19 magnitudes g2d_mag [20][P] as (g2d, g2d_mag): planes 0-9 the same
    sums over |terms|, planes 10-19 sum |term| x its fp32 sensitivity (ges_oracle.c or_render_bwd)."""
    keep = _Keep()
    sp = _splat(pre, keep)
    P = pre["status"].size
    g2d = np.zeros((10, P), np.float64)
    g2d_abs = np.zeros((20, P), np.float64) if with_abs else None
    g = keep(np.ascontiguousarray(dL_dimg, dtype=np.float64))
    mp = None
    if tile_mask is not None:
        tile_mask = keep(np.ascontiguousarray(tile_mask, dtype=np.uint8))
        mp = _ptr(tile_mask, C.c_uint8)
    lst = keep(np.ascontiguousarray(lst if lst.size else np.zeros(1, np.int32), dtype=np.int32))
    rc = lib().or_render_bwd(C.byref(_screen(cam, st)), C.byref(sp), _ptr(offsets, C.c_int64),
                             _ptr(lst, C.c_int32), mp, _ptr(g, C.c_double), _ptr(g2d, C.c_double),
                             _ptr(g2d_abs, C.c_double) if with_abs else None)
    assert rc == 0
    return (g2d, g2d_abs) if with_abs else g2d


def backward_particles(parts, cam, st: Settings, g2d, status=None, flags=None) -> dict:
    """S5b: gradients of the raw parameters (fp64), returned per plane group."""
    keep = _Keep()
    ps = _part_struct(parts, np.float64, keep)
    P, K = parts.P, parts.K
    n_planes = 3 + 3 + 4 + 1 + 3 * K + 1
    out = np.zeros((n_planes, P), np.float64)
    g = keep(np.ascontiguousarray(g2d, dtype=np.float64))
    sp = _ptr(keep(np.ascontiguousarray(status, np.int32)), C.c_int32) if status is not None else None
    fp = _ptr(keep(np.ascontiguousarray(flags, np.int32)), C.c_int32) if flags is not None else None
    lib().or_backward_particles(C.byref(ps), C.byref(_cam(cam)), C.byref(_settings(st)), _ptr(g, C.c_double),
                                sp, fp, _ptr(out, C.c_double))
    return split_planes(out, K)


def grad_magnitude(parts, cam, st: Settings, g2d_abs, status, flags) -> dict:
    """R19: sum over terms of |term| for every parameter gradient entry -- the S5b
    chain evaluated over magnitudes (ges_oracle.c backward_particles_impl,
    absmode) from the S5a magnitudes g2d_abs.  |g| <= bound always; the entry's
    condition number is bound / |g|."""
    keep = _Keep()
    ps = _part_struct(parts, np.float64, keep)
    P, K = parts.P, parts.K
    n_planes = 3 + 3 + 4 + 1 + 3 * K + 1
    out = np.zeros((n_planes, P), np.float64)
    g = keep(np.ascontiguousarray(g2d_abs, dtype=np.float64))
    sp = _ptr(keep(np.ascontiguousarray(status, np.int32)), C.c_int32)
    fp = _ptr(keep(np.ascontiguousarray(flags, np.int32)), C.c_int32)
    lib().or_backward_particles_abs(C.byref(ps), C.byref(_cam(cam)), C.byref(_settings(st)), _ptr(g, C.c_double),
                                    sp, fp, _ptr(out, C.c_double))
    return split_planes(out, K)


def grad_error_scale(parts, cam, st: Settings, g2d, g2d_mag, status, flags) -> dict:
    """R19: first-order error scales of an fp32 evaluation of every parameter
    gradient entry, {"round": ..., "sens": ...}:
        round = sum_j |L_j| g2d_mag[j]  +  S5b_abs(|g2d|)
        sens  = sum_j |L_j| g2d_mag[10 + j]
    L = the per-particle linear map S5b (g2d -> parameter gradients).  round x eps
    bounds the rounding of the pixel sums (|dg2d_j| <= eps sum|terms|) and of the
    chain's own products; sens is how far the fp32 error of the forward alphas
    (and so of every T_k, R18's model) moves the entry.  An entry whose scales are
    large against |g| is ill-conditioned: fp32 arithmetic on either side moves it
    by about eps round + sens, however it is ordered."""
    keep = _Keep()
    ps = _part_struct(parts, np.float64, keep)
    P, K = parts.P, parts.K
    n_planes = 3 + 3 + 4 + 1 + 3 * K + 1
    sp = _ptr(keep(np.ascontiguousarray(status, np.int32)), C.c_int32)
    fp = _ptr(keep(np.ascontiguousarray(flags, np.int32)), C.c_int32)
    c, s = _cam(cam), _settings(st)
    rnd = np.zeros((n_planes, P), np.float64)
    sens = np.zeros((n_planes, P), np.float64)
    out = np.zeros((n_planes, P), np.float64)
    e = np.zeros((10, P), np.float64)
    for j in range(10 if int(st.kernel) == 1 else 9):
        for dst, src_plane in ((rnd, j), (sens, 10 + j)):
            e[:] = 0.0
            e[j] = g2d_mag[src_plane]
            lib().or_backward_particles(C.byref(ps), C.byref(c), C.byref(s), _ptr(e, C.c_double), sp, fp,
                                        _ptr(out, C.c_double))
            dst += np.abs(out)
    e[:] = np.abs(g2d)
    lib().or_backward_particles_abs(C.byref(ps), C.byref(c), C.byref(s), _ptr(e, C.c_double), sp, fp,
                                    _ptr(out, C.c_double))
    rnd += out
    return {"round": split_planes(rnd, K), "sens": split_planes(sens, K)}


def split_planes(flat, K):
    o = 0
    res = {}
    for n, c in (("mean", 3), ("log_scale", 3), ("quat", 4), ("opacity_logit", 1), ("sh", 3 * K), ("beta", 1)):
        res[n] = flat[o:o + c]
        o += c
    res["opacity_logit"] = res["opacity_logit"][0]
    res["beta"] = res["beta"][0]
    return res


# ---------------------------------------------------------------------------
# whole pipeline
# ---------------------------------------------------------------------------
def render(parts, cam, st: Settings, precision: str = "f32", tile_mask=None, membership="rect") -> dict:
    """Definitional forward: S1 in `precision`, membership + depth sort, fp64
    compositing.  Returns the preprocess dict merged with the image outputs."""
    pre = preprocess(parts, cam, st, precision)
    offsets, lst = tile_lists(pre, tile_mask, membership)
    out = render_fwd(pre, cam, st, offsets, lst, tile_mask)
    out.update(pre=pre, offsets=offsets, list=lst)
    return out


def render_and_grad(parts, cam, st: Settings, dL_dimg, precision: str = "f32", tile_mask=None,
                    membership="rect") -> dict:
    """Forward + full backward.  Decisions (visibility, clamps, membership) are
    taken in `precision`; compositing and adjoints are fp64."""
    out = render(parts, cam, st, precision, tile_mask, membership)
    pre = out["pre"]
    g2d = render_bwd(pre, cam, st, out["offsets"], out["list"], dL_dimg, tile_mask)
    grads = backward_particles(parts, cam, st, g2d, pre["status"], pre["flags"])
    out.update(g2d=g2d, grads=grads)
    return out


def loss_f64(parts, cam, st: Settings, dL_dimg) -> float:
    """L = <dL/dimage, image> of the all-fp64 pipeline (for finite differences)."""
    out = render(parts, cam, st, "f64")
    return float(np.sum(out["image"] * dL_dimg))


def log_spec(x) -> np.ndarray:
    """The KEYSPEC natural log (ges_oracle.c or_log_spec), elementwise, x > 1."""
    x = np.ascontiguousarray(x, np.float32)
    y = np.zeros_like(x)
    lib().or_log_spec_array(_ptr(x, C.c_float), _ptr(y, C.c_float), C.c_int64(x.size))
    return y


def exp_spec(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty_like(x)
    lib().or_exp_spec_array(_ptr(x, C.c_float), _ptr(y, C.c_float), C.c_int64(x.size))
    return y


def sh_basis(d, K, precision="f64"):
    if precision == "f64":
        Y = np.zeros(16, np.float64)
        lib().or_sh_basis_f64(C.c_double(d[0]), C.c_double(d[1]), C.c_double(d[2]), C.c_int(K), _ptr(Y, C.c_double))
    else:
        Y = np.zeros(16, np.float32)
        lib().or_sh_basis_f32(C.c_float(d[0]), C.c_float(d[1]), C.c_float(d[2]), C.c_int(K), _ptr(Y, C.c_float))
    return Y[:K]


def set_amb_margin(m: float) -> None:
    """Widen the oracle's decision-ambiguity bound by a relative margin m."""
    lib().or_set_amb_margin(C.c_double(float(m)))
