"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

ctypes marshalling around liboracle.so (oracle/oracle.c, plain sequential C,
-ffp-contract=off).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package; the product
(paper_1812_05540_b200) never does.  See oracle/oracle.h for the citations.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_P = C.POINTER
_I32 = _P(C.c_int32)
_F64 = _P(C.c_double)
_U32 = _P(C.c_uint32)


class Desc(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("uu_rowptr", _I32), ("uu_col", _I32), ("uu_val", _F64),
                ("uf_rowptr", _I32), ("uf_col", _I32), ("uf_val", _F64),
                ("fu_rowptr", _I32), ("fu_col", _I32), ("fu_val", _F64),
                ("ff_rowptr", _I32), ("ff_col", _I32), ("ff_val", _F64),
                ("fs", _F64)]


class Opts(C.Structure):
    _fields_ = [("amg_theta", C.c_double), ("amg_coarse_max", C.c_int), ("amg_max_levels", C.c_int),
                ("zblock", C.c_int), ("tile_x", C.c_int), ("tile_y", C.c_int), ("tile_z", C.c_int),
                ("mech_mode", C.c_int), ("pres_mode", C.c_int), ("local_mode", C.c_int), ("ff_mode", C.c_int),
                ("cpr_mode", C.c_int), ("aps_mode", C.c_int), ("fs_mode", C.c_int), ("rsl_iters", C.c_int),
                ("fs_modulus_scale", C.c_double), ("second_stage", C.c_int), ("local_sweeps", C.c_int),
                ("amg_smoother", C.c_int), ("amg_gs_block", C.c_int), ("amg_cheb_degree", C.c_int),
                ("amg_cheb_lower", C.c_double), ("amg_smoother_p", C.c_int)]


class Phys(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("length", C.c_double), ("nu", C.c_double),
                ("biot", C.c_double), ("gravity", C.c_double), ("rho_w0", C.c_double), ("rho_nw0", C.c_double),
                ("c_w", C.c_double), ("c_nw", C.c_double), ("mu_w", C.c_double), ("mu_nw", C.c_double),
                ("rho_s", C.c_double), ("p0", C.c_double), ("swr", C.c_double), ("snwr", C.c_double),
                ("well_dbhp", C.c_double), ("rw_over_h", C.c_double), ("burden", C.c_int), ("dirichlet_bottom", C.c_int)]


class Info(C.Structure):
    _fields_ = [("iterations", C.c_int), ("restarts", C.c_int), ("status", C.c_int),
                ("est_relres", C.c_double), ("true_relres", C.c_double),
                ("t_setup", C.c_double), ("t_solve", C.c_double)]


def lib():
    global _LIB
    if _LIB is None:
        # ORACLE_OMP=1: the OpenMP build of the same source (timing-only row; bitwise the same results)
        omp = os.environ.get("ORACLE_OMP", "") not in ("", "0")
        path = os.path.join(_HERE, "liboracle_omp.so" if omp else "liboracle.so")
        src = [os.path.join(_HERE, f) for f in os.listdir(_HERE) if f.endswith((".c", ".h"))]
        if not os.path.exists(path) or any(os.path.getmtime(s) > os.path.getmtime(path) for s in src):
            subprocess.check_call(["make", "-s", "-C", os.path.dirname(_HERE), "oracle_omp" if omp else "oracle"])
        L = C.CDLL(path)
        L.orc_default_opts.argtypes = [_P(Opts)]
        L.orc_create.argtypes = [_P(Desc), _P(Opts)]
        L.orc_create.restype = C.c_void_p
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_setup.argtypes = [C.c_void_p]
        L.orc_setup_flow.argtypes = [C.c_void_p, C.c_int]
        L.orc_update_values.argtypes = [C.c_void_p, _P(Desc)]
        L.orc_apply.argtypes = [C.c_void_p, _F64, _F64]
        L.orc_apply_operator.argtypes = [C.c_void_p, _F64, _F64]
        L.orc_solve.argtypes = [C.c_void_p, _F64, _F64, C.c_double, C.c_int, C.c_int, _P(Info)]
        L.orc_richardson.argtypes = [C.c_void_p, _F64, _F64, C.c_double, C.c_int, _P(Info)]
        L.orc_num_levels.argtypes = [C.c_void_p, C.c_int]
        L.orc_level_sizes.argtypes = [C.c_void_p, C.c_int, C.c_int, _P(C.c_int64)]
        L.orc_level_export.argtypes = [C.c_void_p, C.c_int, C.c_int, _I32, _I32, _F64, _I32, _I32, _I32, _F64, _F64]
        L.orc_counters.argtypes = [C.c_void_p, _P(C.c_int64)]
        L.orc_cheb_smooth.argtypes = [C.c_int, _I32, _I32, _F64, C.c_int, C.c_double, _F64, _F64, _F64]
        L.orc_residual.argtypes = [_P(Phys), C.c_double, _F64, _F64, _F64, _F64, _P(C.c_int8), _F64, _F64, _F64]
        L.orc_masses.argtypes = [_P(Phys), _F64, _F64, _F64, _F64, _F64]
        L.orc_porosity.argtypes = [_P(Phys), _F64, _F64, _F64, _F64, _F64]
        L.orc_get_spp.argtypes = [C.c_void_p, _F64, _I32, _I32, _F64]
        L.orc_get_cpr.argtypes = [C.c_void_p, _F64, _F64, _F64]
        L.orc_mis2.argtypes = [C.c_int, _I32, _I32, _U32, C.c_int, _I32, _P(C.c_int)]
        L.orc_amg_build.argtypes = [C.c_int, C.c_int, _I32, _I32, _F64, _I32, _P(Opts)]
        L.orc_amg_build.restype = C.c_void_p
        L.orc_amg_vcycle.argtypes = [C.c_void_p, _F64, _F64]
        L.orc_amg_levels.argtypes = [C.c_void_p]
        L.orc_amg_level_sizes.argtypes = [C.c_void_p, C.c_int, _P(C.c_int64)]
        L.orc_amg_level_export.argtypes = [C.c_void_p, C.c_int, _I32, _I32, _F64, _I32, _I32, _I32, _F64, _F64]
        L.orc_amg_free.argtypes = [C.c_void_p]
        L.orc_amg_level_detail.argtypes = [C.c_void_p, C.c_int, _I32, _I32, _F64]
        L.orc_amg_level_colour.argtypes = [C.c_void_p, C.c_int, _I32]
        L.orc_amg_level_gs.argtypes = [C.c_void_p, C.c_int, _F64]
        L.orc_amg_build_coloured.argtypes = [C.c_int, C.c_int, _I32, _I32, _F64, _I32, _I32, _P(Opts)]
        L.orc_amg_build_coloured.restype = C.c_void_p
        L.orc_level_colour.argtypes = [C.c_void_p, C.c_int, C.c_int, _I32]
        L.orc_strength.argtypes = [C.c_int, C.c_int, _I32, _I32, _F64, _I32, C.c_double, _P(C.c_uint8)]
        L.orc_ilu_build.argtypes = [C.c_int] * 6 + [_I32, _I32, _F64]
        L.orc_ilu_build.restype = C.c_void_p
        L.orc_ilu_apply.argtypes = [C.c_void_p, _F64, _F64]
        L.orc_ilu_free.argtypes = [C.c_void_p]
        L.orc_bgs_build.argtypes = [C.c_int] * 6 + [_I32, _I32, _F64]
        L.orc_bgs_build.restype = C.c_void_p
        L.orc_bgs_apply.argtypes = [C.c_void_p, _F64, _F64]
        _LIB = L
    return _LIB


def _p(a):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    if a.dtype == np.int32:
        return a.ctypes.data_as(_I32)
    if a.dtype == np.uint32:
        return a.ctypes.data_as(_U32)
    assert a.dtype == np.float64, a.dtype
    return a.ctypes.data_as(_F64)


def default_opts(**kw) -> Opts:
    o = Opts()
    lib().orc_default_opts(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def _export(sizes_fn, export_fn, lvl):
    out = (C.c_int64 * 6)()
    sizes_fn(lvl, out)
    n, nnz, nagg, pnz, nc, coarsest = list(out)
    d = dict(n=n, nnz=nnz, nagg=nagg, nc=nc, coarsest=bool(coarsest))
    d["A_rp"] = np.empty(n + 1, np.int32)
    d["A_ci"] = np.empty(nnz, np.int32)
    d["A_v"] = np.empty((nnz, nc))
    d["dl1"] = np.empty((n, nc))
    if not coarsest:
        d["agg"] = np.empty(n, np.int32)
        d["P_rp"] = np.empty(n + 1, np.int32)
        d["P_ci"] = np.empty(pnz, np.int32)
        d["P_v"] = np.empty((pnz, nc))
    export_fn(lvl, _p(d["A_rp"]), _p(d["A_ci"]), _p(d["A_v"]), _p(d.get("agg")), _p(d.get("P_rp")),
              _p(d.get("P_ci")), _p(d.get("P_v")), _p(d["dl1"]))
    return d


class Oracle:
    """One coupled problem (synth.Problem) with the oracle's setup products."""

    def __init__(self, pb, **opts):
        self.pb = pb
        self._keep = [np.ascontiguousarray(x) for x in (
            pb.uu_rowptr, pb.uu_col, pb.uu_val, pb.uf_rowptr, pb.uf_col, pb.uf_val,
            pb.fu_rowptr, pb.fu_col, pb.fu_val, pb.ff_rowptr, pb.ff_col, pb.ff_val, pb.fs)]
        k = self._keep
        d = Desc(pb.nx, pb.ny, pb.nz, *[_p(x) for x in k])
        self.opts = default_opts(**opts)
        self.h = lib().orc_create(C.byref(d), C.byref(self.opts))
        self.n = pb.n

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().orc_destroy(self.h)
            except TypeError:       # interpreter shutdown: the module globals are already gone
                pass
            self.h = None

    def setup(self):
        rc = lib().orc_setup(self.h)
        if rc != 0:
            raise RuntimeError(f"orc_setup failed ({rc})")
        return self

    def update_values(self, pb):
        """A Newton step's new values on the same patterns (orc_update_values)."""
        keep = [np.ascontiguousarray(x) for x in (
            pb.uu_rowptr, pb.uu_col, pb.uu_val, pb.uf_rowptr, pb.uf_col, pb.uf_val,
            pb.fu_rowptr, pb.fu_col, pb.fu_val, pb.ff_rowptr, pb.ff_col, pb.ff_val, pb.fs)]
        d = Desc(pb.nx, pb.ny, pb.nz, *[_p(x) for x in keep])
        if lib().orc_update_values(self.h, C.byref(d)) != 0:
            raise ValueError("orc_update_values: the patterns changed")
        return self

    def setup_flow(self, refresh=False):
        rc = lib().orc_setup_flow(self.h, int(refresh))
        if rc != 0:
            raise RuntimeError(f"orc_setup_flow failed ({rc})")
        return self

    def apply(self, v):
        v = np.ascontiguousarray(v, np.float64)
        z = np.zeros(self.n)
        rc = lib().orc_apply(self.h, _p(v), _p(z))
        if rc != 0:
            raise RuntimeError(f"orc_apply failed ({rc})")
        return z

    def operator(self, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.n)
        lib().orc_apply_operator(self.h, _p(x), _p(y))
        return y

    def solve(self, b, rtol=1e-8, m=64, maxit=1000):
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(self.n)
        info = Info()
        lib().orc_solve(self.h, _p(b), _p(x), rtol, m, maxit, C.byref(info))
        return x, dict(iterations=info.iterations, restarts=info.restarts, status=info.status,
                       est_relres=info.est_relres, true_relres=info.true_relres, t_solve=info.t_solve)

    def richardson(self, b, rtol=1e-8, maxit=1000):
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(self.n)
        info = Info()
        lib().orc_richardson(self.h, _p(b), _p(x), rtol, maxit, C.byref(info))
        return x, dict(iterations=info.iterations, status=info.status, true_relres=info.true_relres)

    def num_levels(self, which):
        return lib().orc_num_levels(self.h, which)

    def level(self, which, lvl):
        L = lib()
        return _export(lambda l, o: L.orc_level_sizes(self.h, which, l, o),
                       lambda l, *a: L.orc_level_export(self.h, which, l, *a), lvl)

    def hierarchy(self, which):
        return [self.level(which, l) for l in range(self.num_levels(which))]

    def colour(self, which, lvl):
        n = self.level(which, lvl)["n"]
        col = np.empty(n, np.int32)
        nc = lib().orc_level_colour(self.h, which, lvl, _p(col))
        return col, nc

    def counters(self):
        out = (C.c_int64 * 4)()
        lib().orc_counters(self.h, out)
        return dict(skipped_dss=out[0], perturbed=out[1], fallbacks=out[2])

    def spp(self):
        pb = self.pb
        nnz = int(pb.ff_rowptr[-1])
        Dss = np.empty(pb.Nc)
        rp = np.empty(pb.Nc + 1, np.int32)
        ci = np.empty(nnz, np.int32)
        v = np.empty(nnz)
        lib().orc_get_spp(self.h, _p(Dss), _p(rp), _p(ci), _p(v))
        return Dss, rp, ci, v

    def cpr(self):
        """(D_ss^(CPR), D_ps^(CPR), D_fs used by a1 as (Nc, 2))."""
        Nc = self.pb.Nc
        Dss, Dps, fs = np.empty(Nc), np.empty(Nc), np.empty(2 * Nc)
        lib().orc_get_cpr(self.h, _p(Dss), _p(Dps), _p(fs))
        return Dss, Dps, fs.reshape(Nc, 2)


def mis2(rp, ci, hashes, rounds=False):
    n = len(rp) - 1
    st = np.empty(n, np.int32)
    nr = C.c_int(0)
    lib().orc_mis2(n, _p(np.ascontiguousarray(rp, np.int32)), _p(np.ascontiguousarray(ci, np.int32)),
                   _p(np.ascontiguousarray(hashes, np.uint32)), int(rounds), _p(st), C.byref(nr))
    return st, nr.value


def strength(rp, ci, v, zb, theta=0.25):
    """Symmetrised strength flags (one per stored entry) of R-strength."""
    n = len(rp) - 1
    v = np.ascontiguousarray(v, np.float64)
    nc = 1 if v.ndim == 1 else v.shape[1]
    E = np.zeros(int(rp[-1]), np.uint8)
    rc = lib().orc_strength(n, nc, _p(np.ascontiguousarray(rp, np.int32)), _p(np.ascontiguousarray(ci, np.int32)), _p(v),
                            _p(np.ascontiguousarray(zb, np.int32)), theta, E.ctypes.data_as(_P(C.c_uint8)))
    if rc != 0:
        raise ValueError("pattern not structurally symmetric")
    return E.astype(bool)


def fmix32(x):
    x = np.asarray(x, np.uint64) & 0xFFFFFFFF
    x ^= x >> 16
    x = (x * 0x85EBCA6B) & 0xFFFFFFFF
    x ^= x >> 13
    x = (x * 0xC2B2AE35) & 0xFFFFFFFF
    x ^= x >> 16
    return x.astype(np.uint32)


def phys(params):
    """orc_phys from a synth parameter dict (synth.params_of)."""
    return Phys(**{k: params[k] for k, _ in Phys._fields_})


def _f64(a):
    return np.ascontiguousarray(a, np.float64)


def residual(params, fields, x, mprev, dt):
    """r(x) of Appendix B.1 (raw units; x = [u | (s, p [Pa])]); fields: E, perm, phi0, pref, well."""
    P = phys(params)
    keep = [_f64(fields[k]) for k in ("E", "perm", "phi0", "pref")] + [_f64(x), _f64(mprev)]
    w = np.ascontiguousarray(fields["well"], np.int8) if fields.get("well") is not None else None
    R = np.empty(len(x))
    rc = lib().orc_residual(C.byref(P), float(dt), *(_p(a) for a in keep[:4]),
                            w.ctypes.data_as(_P(C.c_int8)) if w is not None else None, _p(keep[4]), _p(keep[5]), _p(R))
    if rc:
        raise ValueError("orc_residual failed")
    return R


def masses(params, fields, x):
    P = phys(params)
    keep = [_f64(fields[k]) for k in ("E", "phi0", "pref")] + [_f64(x)]
    m = np.empty(2 * params["nx"] * params["ny"] * params["nz"])
    lib().orc_masses(C.byref(P), *(_p(a) for a in keep), _p(m))
    return m


def porosity(params, fields, x):
    P = phys(params)
    keep = [_f64(fields[k]) for k in ("E", "phi0", "pref")] + [_f64(x)]
    phi = np.empty(params["nx"] * params["ny"] * params["nz"])
    lib().orc_porosity(C.byref(P), *(_p(a) for a in keep), _p(phi))
    return phi


def cheb_smooth(rp, ci, v, b, x0=None, degree=2, lower=0.3):
    """R-cheb: `degree` Chebyshev steps on D_l1^-1 A (scalar CSR) from x0 (None = 0)."""
    n = len(rp) - 1
    keep = [np.ascontiguousarray(rp, np.int32), np.ascontiguousarray(ci, np.int32), np.ascontiguousarray(v, np.float64),
            np.ascontiguousarray(b, np.float64), None if x0 is None else np.ascontiguousarray(x0, np.float64)]
    x = np.empty(n)
    if lib().orc_cheb_smooth(n, _p(keep[0]), _p(keep[1]), _p(keep[2]), degree, lower, _p(keep[3]), _p(keep[4]), _p(x)):
        raise ValueError("orc_cheb_smooth: bad degree / interval")
    return x


class Amg:
    """Standalone oracle AMG on a (multi-component) CSR matrix, for pins."""

    def __init__(self, rp, ci, v, zb=None, colour0=None, **opts):
        self.n = len(rp) - 1
        v = np.ascontiguousarray(v, np.float64)
        self.nc = 1 if v.ndim == 1 else v.shape[1]
        zb = np.zeros(self.n, np.int32) if zb is None else np.ascontiguousarray(zb, np.int32)
        o = default_opts(**opts)
        self._keep = (np.ascontiguousarray(rp, np.int32), np.ascontiguousarray(ci, np.int32), v, zb,
                      None if colour0 is None else np.ascontiguousarray(colour0, np.int32))
        self.h = lib().orc_amg_build_coloured(self.n, self.nc, _p(self._keep[0]), _p(self._keep[1]), _p(v), _p(zb),
                                              _p(self._keep[4]), C.byref(o))
        if not self.h:
            raise RuntimeError("orc_amg_build failed")

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_amg_free(self.h)
            self.h = None

    def vcycle(self, b):
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros_like(b)
        lib().orc_amg_vcycle(self.h, _p(b), _p(x))
        return x

    def colour(self, lvl):
        """(colour per row, number of colours) of a level's GS smoother (R-gs)."""
        n = self.levels()[lvl]["n"]
        col = np.empty(n, np.int32)
        nc = lib().orc_amg_level_colour(self.h, lvl, _p(col))
        return col, nc

    def gs(self, lvl):
        """(gs_block of the level -- 0 for multicolour --, hybrid l1 diagonal (n, nc)) of the GS smoother."""
        n = self.levels()[lvl]["n"]
        dh = np.zeros((n, self.nc))
        return lib().orc_amg_level_gs(self.h, lvl, _p(dh)), dh

    def detail(self, lvl):
        """(MIS(2) state, phase-1 aggregate ids, omega per component) of a non-coarsest level."""
        n = self.levels()[lvl]["n"]
        st, ph1, om = np.empty(n, np.int32), np.empty(n, np.int32), np.empty(self.nc)
        if lib().orc_amg_level_detail(self.h, lvl, _p(st), _p(ph1), _p(om)) != 0:
            raise ValueError(f"level {lvl} is the coarsest")
        return st, ph1, om

    def levels(self):
        L = lib()
        nl = L.orc_amg_levels(self.h)
        return [_export(lambda l, o: L.orc_amg_level_sizes(self.h, l, o),
                        lambda l, *a: L.orc_amg_level_export(self.h, l, *a), l) for l in range(nl)]


class Ilu:
    """Standalone oracle tile ILU(0) on an interleaved 2x2 BSR cell matrix, for pins."""

    def __init__(self, nx, ny, nz, tile, rp, ci, v):
        self._keep = (np.ascontiguousarray(rp, np.int32), np.ascontiguousarray(ci, np.int32),
                      np.ascontiguousarray(v, np.float64))
        self.h = lib().orc_ilu_build(nx, ny, nz, tile[0], tile[1], tile[2], *[_p(x) for x in self._keep])

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_ilu_free(self.h)
            self.h = None

    def apply(self, w):
        w = np.ascontiguousarray(w, np.float64)
        dz = np.zeros_like(w)
        lib().orc_ilu_apply(self.h, _p(w), _p(dz))
        return dz


class Bgs(Ilu):
    """Standalone oracle hybrid block Gauss-Seidel sweep (tile = processor), for pins."""

    def __init__(self, nx, ny, nz, tile, rp, ci, v):
        self._keep = (np.ascontiguousarray(rp, np.int32), np.ascontiguousarray(ci, np.int32),
                      np.ascontiguousarray(v, np.float64))
        self.h = lib().orc_bgs_build(nx, ny, nz, tile[0], tile[1], tile[2], *[_p(x) for x in self._keep])

    def apply(self, w):
        w = np.ascontiguousarray(w, np.float64)
        dz = np.zeros_like(w)
        lib().orc_bgs_apply(self.h, _p(w), _p(dz))
        return dz
