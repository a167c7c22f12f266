"""Seeded synthetic inputs for the two-stage preconditioner path.

This module is the ONLY thing the oracle side and the CUDA side share: it
generates one linearised coupled poromechanics Jacobian (block layout of
include/tsp.h) at a synthetic state, plus x_rand and b = A x_rand.  It holds
none of the preconditioner / FGMRES arithmetic.  The physics is cited in
synth/synth.c; the field recipes follow BASELINE.json configs[0..4] with the
readings listed in DESIGN.md.

Plain ctypes marshalling around libsynth.so (built by `make synth`).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class Params(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("recipe", C.c_int),
        ("seed", C.c_uint64),
        ("E_median", C.c_double), ("E_sigma", C.c_double),
        ("perm_median", C.c_double), ("perm_sigma", C.c_double),
        ("nu", C.c_double), ("biot", C.c_double), ("gravity", C.c_double), ("dt", C.c_double),
        ("rho_w0", C.c_double), ("rho_nw0", C.c_double), ("c_w", C.c_double), ("c_nw", C.c_double),
        ("mu_w", C.c_double), ("mu_nw", C.c_double), ("rho_s", C.c_double), ("p0", C.c_double),
        ("swr", C.c_double), ("snwr", C.c_double),
        ("well_dbhp", C.c_double), ("rw_over_h", C.c_double), ("state_dp", C.c_double), ("p_unit", C.c_double), ("length", C.c_double),
        ("wells", C.c_int), ("dirichlet_bottom", C.c_int), ("row_scale", C.c_int),
        ("burden", C.c_int), ("well_pattern", C.c_int), ("pad2_", C.c_int),
        ("burden_perm", C.c_double), ("burden_phi", C.c_double),
    ]


_P = C.POINTER
_I32 = _P(C.c_int32)
_F64 = _P(C.c_double)


class Out(C.Structure):
    _fields_ = [
        ("uu_rowptr", _I32), ("uu_col", _I32), ("uu_val", _F64),
        ("uf_rowptr", _I32), ("uf_col", _I32), ("uf_val", _F64),
        ("fu_rowptr", _I32), ("fu_col", _I32), ("fu_val", _F64),
        ("ff_rowptr", _I32), ("ff_col", _I32), ("ff_val", _F64),
        ("fs", _F64), ("x_rand", _F64), ("b", _F64),
        ("E", _F64), ("perm", _F64), ("phi", _F64), ("sat", _F64), ("pres", _F64),
        ("scales", _F64),
    ]


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(path):
            import subprocess
            subprocess.check_call(["make", "-s", "-C", os.path.dirname(_HERE), "synth"])
        _LIB = C.CDLL(path)
        _LIB.synth_sizes.argtypes = [_P(Params), _P(C.c_int64)]
        _LIB.synth_generate.argtypes = [_P(Params), _P(Out)]
        _LIB.synth_generate.restype = C.c_int
        _LIB.synth_fields.argtypes = [_P(Params)] + [_F64] * 6 + [_P(C.c_int8)]
        _LIB.synth_fields.restype = C.c_int
        _LIB.synth_assemble_state.argtypes = [_P(Params)] + [_F64] * 6 + [_P(Out)]
        _LIB.synth_assemble_state.restype = C.c_int
    return _LIB


# Constants absent from BASELINE.json come from Table 1 in SI units.
DEFAULTS = dict(
    E_median=1e9, E_sigma=0.5, perm_median=1e-13, perm_sigma=1.0,
    nu=0.25, biot=1.0, gravity=9.81, dt=86400.0,
    rho_w0=1035.0, rho_nw0=863.0, c_w=4.34e-10, c_nw=1.98e-10,
    mu_w=1e-3, mu_nw=5e-3, rho_s=2650.0, p0=1e7, swr=0.2, snwr=0.2,
    well_dbhp=5e6, rw_over_h=0.1, state_dp=0.0, p_unit=1e6, length=10000.0, wells=1, dirichlet_bottom=1, row_scale=1,
    seed=0, recipe=1, burden=0, well_pattern=0, burden_perm=1e-17, burden_phi=0.01,
)

# BASELINE.json configs[0..4] (C1..C5); recipes per SURVEY D17.
CONFIGS = {
    "C1": dict(nx=8, ny=8, nz=8, recipe=1, perm_sigma=1.0),
    "C2": dict(nx=32, ny=32, nz=32, recipe=2, perm_sigma=2.0),
    "C3": dict(nx=64, ny=64, nz=64, recipe=3, perm_sigma=3.0),
    "C4": dict(nx=128, ny=128, nz=64, recipe=4, perm_sigma=2.0),
    "C5": dict(nx=256, ny=256, nz=128, recipe=5, perm_sigma=2.0),
}
# Second workload (SURVEY NEXT-f4 ii, DESIGN.md R-s10): the SPE10-based example's shape -- 60 x 220 x 252 cells,
# 0.01 mD / 1 % over- and underburden, homogeneous E = 5000 MPa, nu = 0.25, five wells -- with the
# correlated generator (D17) in the 84 reservoir layers, since the SPE10 data are not available.
_STAIR = dict(recipe=6, E_median=5e9, E_sigma=0.0, mu_w=3e-4, mu_nw=3e-3, well_pattern=2)
WORKLOADS = {
    # Staircase benchmark (SURVEY NEXT-f4 i, DESIGN.md R-stair): Table 1's staircase column on the four grids of
    # Table 2 (levels 2 and 3 are the C4 and C5 grids), channel geometry by the documented convention
    "ST0": dict(nx=32, ny=32, nz=16, **_STAIR),
    "ST1": dict(nx=64, ny=64, nz=32, **_STAIR),
    "ST2": dict(nx=128, ny=128, nz=64, **_STAIR),
    "ST3": dict(nx=256, ny=256, nz=128, **_STAIR),
    "S10": dict(nx=60, ny=220, nz=252, recipe=4, perm_median=1e-14, perm_sigma=3.0, E_median=5e9, E_sigma=0.0,
                burden=84, well_pattern=1),   # cells 167 m: the R-geom convention (normalised 10 km domain side)
}


@dataclass
class Problem:
    nx: int
    ny: int
    nz: int
    params: dict
    uu_rowptr: np.ndarray
    uu_col: np.ndarray
    uu_val: np.ndarray      # (B_uu, 3, 3)
    uf_rowptr: np.ndarray
    uf_col: np.ndarray
    uf_val: np.ndarray      # (B_uf, 3, 2)
    fu_rowptr: np.ndarray
    fu_col: np.ndarray
    fu_val: np.ndarray      # (B_fu, 2, 3)
    ff_rowptr: np.ndarray
    ff_col: np.ndarray
    ff_val: np.ndarray      # (B_ff, 2, 2)
    fs: np.ndarray          # (N_c, 2): D_sp, D_pp (row-scaled)
    x_rand: np.ndarray
    b: np.ndarray
    fields: dict = field(default_factory=dict)
    scales: np.ndarray = None

    @property
    def Nn(self):
        return (self.nx + 1) * (self.ny + 1) * (self.nz + 1)

    @property
    def Nc(self):
        return self.nx * self.ny * self.nz

    @property
    def n(self):
        return 3 * self.Nn + 2 * self.Nc


def sizes(nx, ny, nz):
    p = Params(nx=nx, ny=ny, nz=nz)
    out = (C.c_int64 * 8)()
    _lib().synth_sizes(C.byref(p), out)
    return dict(Nn=out[0], Nc=out[1], Buu=out[2], Buf=out[3], Bfu=out[4], Bff=out[5], n=out[6], faces=out[7])


def generate(config: str | None = None, **overrides) -> Problem:
    """Generate one coupled Jacobian.  `config` is C1..C5 (BASELINE.json
    configs[0..4]); keyword overrides change any Params field (e.g. nx=3, biot=0)."""
    kw = dict(DEFAULTS)
    if config is not None:
        kw.update(CONFIGS[config] if config in CONFIGS else WORKLOADS[config])
    kw.update(overrides)
    p = Params(**{k: v for k, v in kw.items() if k in dict(Params._fields_)})
    s = sizes(p.nx, p.ny, p.nz)
    Nn, Nc = s["Nn"], s["Nc"]
    a = dict(
        uu_rowptr=np.empty(Nn + 1, np.int32), uu_col=np.empty(s["Buu"], np.int32), uu_val=np.empty((s["Buu"], 3, 3)),
        uf_rowptr=np.empty(Nn + 1, np.int32), uf_col=np.empty(s["Buf"], np.int32), uf_val=np.empty((s["Buf"], 3, 2)),
        fu_rowptr=np.empty(Nc + 1, np.int32), fu_col=np.empty(s["Bfu"], np.int32), fu_val=np.empty((s["Bfu"], 2, 3)),
        ff_rowptr=np.empty(Nc + 1, np.int32), ff_col=np.empty(s["Bff"], np.int32), ff_val=np.empty((s["Bff"], 2, 2)),
        fs=np.empty((Nc, 2)), x_rand=np.empty(s["n"]), b=np.empty(s["n"]),
    )
    f = {k: np.empty(Nc) for k in ("E", "perm", "phi", "sat", "pres")}
    scales = np.empty(3)

    def ptr(x):
        return x.ctypes.data_as(_I32 if x.dtype == np.int32 else _F64)

    o = Out(**{k: ptr(v) for k, v in a.items()}, **{k: ptr(v) for k, v in f.items()}, scales=ptr(scales))
    rc = _lib().synth_generate(C.byref(p), C.byref(o))
    if rc != 0:
        raise ValueError(f"synth_generate failed ({rc})")
    return Problem(nx=p.nx, ny=p.ny, nz=p.nz, params=kw, fields=f, scales=scales, **a)


def params_of(config: str | None = None, **overrides) -> dict:
    """The full parameter set of a config (DEFAULTS < config < overrides)."""
    kw = dict(DEFAULTS)
    if config is not None:
        kw.update(CONFIGS[config] if config in CONFIGS else WORKLOADS[config])
    kw.update(overrides)
    return kw


def fields(config: str | None = None, x_rand: bool = True, **overrides) -> dict:
    """The per-cell state of `generate` (E, perm, phi, sat, pres; same seeded streams, same values), the well
    perforation of each cell (0 none, 1 injector, 2 producer) and x_rand,
    WITHOUT assembling the Jacobian: the input of the GPU assembly (tsp_assemble)."""
    kw = params_of(config, **overrides)
    p = Params(**{k: v for k, v in kw.items() if k in dict(Params._fields_)})
    s = sizes(p.nx, p.ny, p.nz)
    f = {k: np.empty(s["Nc"]) for k in ("E", "perm", "phi", "sat", "pres")}
    xr = np.empty(s["n"]) if x_rand else None
    f["well"] = np.empty(s["Nc"], np.int8)
    rc = _lib().synth_fields(C.byref(p), *(f[k].ctypes.data_as(_F64) for k in ("E", "perm", "phi", "sat", "pres")),
                             xr.ctypes.data_as(_F64) if xr is not None else None, f["well"].ctypes.data_as(_P(C.c_int8)))
    if rc != 0:
        raise ValueError(f"synth_fields failed ({rc})")
    f["x_rand"] = xr
    f["params"] = kw
    return f


def assemble_state(params: dict, E, perm, phi, sat, pres, phi0=None) -> Problem:
    """The Jacobian blocks at a given state (synth_assemble_state: the CPU assembler at arbitrary fields; phi the
    porosity at the state, phi0 the reference porosity of eq:linearized_porosity, pres in Pa).  x_rand and b are
    not produced (zeros)."""
    p = Params(**{k: v for k, v in params.items() if k in dict(Params._fields_)})
    s = sizes(p.nx, p.ny, p.nz)
    Nn, Nc = s["Nn"], s["Nc"]
    a = dict(
        uu_rowptr=np.empty(Nn + 1, np.int32), uu_col=np.empty(s["Buu"], np.int32), uu_val=np.empty((s["Buu"], 3, 3)),
        uf_rowptr=np.empty(Nn + 1, np.int32), uf_col=np.empty(s["Buf"], np.int32), uf_val=np.empty((s["Buf"], 3, 2)),
        fu_rowptr=np.empty(Nc + 1, np.int32), fu_col=np.empty(s["Bfu"], np.int32), fu_val=np.empty((s["Bfu"], 2, 3)),
        ff_rowptr=np.empty(Nc + 1, np.int32), ff_col=np.empty(s["Bff"], np.int32), ff_val=np.empty((s["Bff"], 2, 2)),
        fs=np.empty((Nc, 2)), x_rand=np.zeros(s["n"]), b=np.zeros(s["n"]),
    )
    f = {k: np.ascontiguousarray(v, np.float64) for k, v in dict(E=E, perm=perm, phi=phi, sat=sat, pres=pres).items()}
    f0 = np.ascontiguousarray(phi0, np.float64) if phi0 is not None else None
    scales = np.empty(3)

    def ptr(x):
        return x.ctypes.data_as(_I32 if x.dtype == np.int32 else _F64)

    o = Out(**{k: ptr(v) for k, v in a.items()}, **{k: ptr(np.empty(Nc)) for k in ("E", "perm", "phi", "sat", "pres")},
            scales=ptr(scales))
    rc = _lib().synth_assemble_state(C.byref(p), *(ptr(f[k]) for k in ("E", "perm", "phi")),
                                     ptr(f0) if f0 is not None else None, ptr(f["sat"]), ptr(f["pres"]), C.byref(o))
    if rc != 0:
        raise ValueError(f"synth_assemble_state failed ({rc})")
    return Problem(nx=p.nx, ny=p.ny, nz=p.nz, params=dict(params), fields=f, scales=scales, **a)


def to_scipy(pb: Problem):
    """Assemble the full coupled matrix in natural [u | f] order as scipy CSR
    (test infrastructure for pins; interleaved f = (s_K, p_K))."""
    import scipy.sparse as sp

    A_uu = sp.bsr_matrix((pb.uu_val, pb.uu_col, pb.uu_rowptr), shape=(3 * pb.Nn, 3 * pb.Nn))
    A_uf = sp.bsr_matrix((pb.uf_val, pb.uf_col, pb.uf_rowptr), shape=(3 * pb.Nn, 2 * pb.Nc))
    A_fu = sp.bsr_matrix((pb.fu_val, pb.fu_col, pb.fu_rowptr), shape=(2 * pb.Nc, 3 * pb.Nn))
    A_ff = sp.bsr_matrix((pb.ff_val, pb.ff_col, pb.ff_rowptr), shape=(2 * pb.Nc, 2 * pb.Nc))
    return sp.bmat([[A_uu, A_uf], [A_fu, A_ff]]).tocsr(), (A_uu, A_uf, A_fu, A_ff)


def slab_partition(nx, ny, nz, zblock, rank, nranks):
    """The z-slab partition of include/tsp.h (rank r owns z-blocks
    [floor(r nzb / P), floor((r+1) nzb / P))): returns (k0, k1, node0, nnodes,
    cell0, ncells).  tests/test_multirank_cpu.py pins it against tsp_partition."""
    nzb = (nz + zblock - 1) // zblock
    zlo, zhi = rank * nzb // nranks, (rank + 1) * nzb // nranks
    k0, k1 = zlo * zblock, min(zhi * zblock, nz)
    NP, CP = (nx + 1) * (ny + 1), nx * ny
    last = int(rank == nranks - 1)
    return k0, k1, k0 * NP, (k1 - k0 + last) * NP, k0 * CP, (k1 - k0) * CP


@dataclass
class LocalProblem:
    """The rows one rank owns (GLOBAL column ids) -- what a rank passes to tsp_create."""
    nx: int
    ny: int
    nz: int
    rank: int
    nranks: int
    node0: int
    cell0: int
    uu_rowptr: np.ndarray
    uu_col: np.ndarray
    uu_val: np.ndarray
    uf_rowptr: np.ndarray
    uf_col: np.ndarray
    uf_val: np.ndarray
    fu_rowptr: np.ndarray
    fu_col: np.ndarray
    fu_val: np.ndarray
    ff_rowptr: np.ndarray
    ff_col: np.ndarray
    ff_val: np.ndarray
    fs: np.ndarray
    Nn: int
    Nc: int

    @property
    def n(self):
        return 3 * self.Nn + 2 * self.Nc

    def local(self, v, nn_glob):
        """This rank's part [u_own | f_own] of a global vector [u | f]."""
        return np.concatenate([v[3 * self.node0:3 * (self.node0 + self.Nn)],
                               v[3 * nn_glob + 2 * self.cell0:3 * nn_glob + 2 * (self.cell0 + self.Nc)]])


def _rows(rp, ci, v, r0, nr):
    a, b = rp[r0], rp[r0 + nr]
    # copies: a rank's slab must not keep the global arrays alive (bench.py frees them)
    return (rp[r0:r0 + nr + 1] - a).astype(np.int32), ci[a:b].copy(), v[a:b].copy()


def local_problem(pb: Problem, rank: int, nranks: int, zblock: int = 16) -> LocalProblem:
    k0, k1, n0, nn, c0, ncl = slab_partition(pb.nx, pb.ny, pb.nz, zblock, rank, nranks)
    d = {}
    for name, r0, nr in (("uu", n0, nn), ("uf", n0, nn), ("fu", c0, ncl), ("ff", c0, ncl)):
        rp, ci, v = _rows(getattr(pb, name + "_rowptr"), getattr(pb, name + "_col"), getattr(pb, name + "_val"), r0, nr)
        d[name + "_rowptr"], d[name + "_col"], d[name + "_val"] = rp, ci, v
    return LocalProblem(nx=pb.nx, ny=pb.ny, nz=pb.nz, rank=rank, nranks=nranks, node0=n0, cell0=c0,
                        fs=pb.fs[c0:c0 + ncl].copy(), Nn=nn, Nc=ncl, **d)
