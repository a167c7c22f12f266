"""Thin ctypes binding of libtsp.so (include/tsp.h).  Argument marshalling only:
every step of the preconditioner / solver runs in the CUDA kernels of the
library.  There is no CPU fallback: if libtsp.so is missing or no CUDA device
is present, the calls raise.

Names follow the C-ABI: tsp_create, tsp_setup, tsp_apply_preconditioner,
tsp_apply_operator, tsp_solve, tsp_get_stats, tsp_export_level, ...
`Tsp` bundles them for a synth.Problem-like input.
"""
from __future__ import annotations

import ctypes as C
import atexit
import os
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSP_LIB_DEV") or os.path.join(_HERE, "libtsp.so")   # TSP_LIB_DEV: developer A/B builds only
_LIB = None
_P = C.POINTER

TSP_SETUP_MECH = 1
TSP_SETUP_FLOW = 2
TSP_SETUP_REFRESH = 4     # with TSP_SETUP_FLOW: frozen-aggregation value refresh after update_values (NEXT-f1)
STATUS = {0: "OK", 1: "NOT_CONVERGED", -1: "INVALID_ARG", -2: "DIM_MISMATCH", -3: "STATE", -4: "CUDA",
          -5: "NCCL", -6: "OOM", -7: "SINGULAR", -8: "NUMERIC"}


class tsp_options(C.Structure):
    _fields_ = [("amg_theta", C.c_double), ("amg_coarse_max", C.c_int), ("amg_max_levels", C.c_int),
                ("zblock", C.c_int), ("tile_x", C.c_int), ("tile_y", C.c_int), ("tile_z", C.c_int),
                ("replicate_rows", C.c_int), ("cpr_mode", C.c_int), ("aps_mode", C.c_int), ("fs_mode", C.c_int),
                ("rsl_iters", C.c_int), ("fs_modulus_scale", C.c_double), ("second_stage", C.c_int),
                ("local_sweeps", C.c_int), ("amg_smoother", C.c_int), ("amg_gs_block", C.c_int),
                ("amg_cheb_degree", C.c_int), ("amg_cheb_lower", C.c_double), ("amg_smoother_p", C.c_int)]


class tsp_bsr(C.Structure):
    _fields_ = [("rowptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p)]


class tsp_asm_params(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("length", C.c_double),
                ("nu", C.c_double), ("biot", C.c_double), ("gravity", C.c_double), ("dt", C.c_double),
                ("rho_w0", C.c_double), ("rho_nw0", C.c_double), ("c_w", C.c_double), ("c_nw", C.c_double),
                ("mu_w", C.c_double), ("mu_nw", C.c_double), ("rho_s", C.c_double), ("p0", C.c_double),
                ("swr", C.c_double), ("snwr", C.c_double), ("well_dbhp", C.c_double), ("rw_over_h", C.c_double),
                ("p_unit", C.c_double), ("burden", C.c_int), ("dirichlet_bottom", C.c_int), ("row_scale", C.c_int)]


class tsp_cell_fields(C.Structure):
    _fields_ = [("E", C.c_void_p), ("perm", C.c_void_p), ("phi", C.c_void_p), ("sat", C.c_void_p),
                ("pres", C.c_void_p), ("well", C.c_void_p), ("phi0", C.c_void_p)]


class tsp_bsr_out(C.Structure):
    _fields_ = [("rowptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p)]


class tsp_newton_opts(C.Structure):
    _fields_ = [("rtol", C.c_double), ("atol", C.c_double), ("max_newton", C.c_int), ("lin_rtol", C.c_double),
                ("max_lin_iters", C.c_int), ("refresh", C.c_int), ("max_halvings", C.c_int)]


class tsp_newton_info(C.Structure):
    _fields_ = [("newton_iters", C.c_int), ("lin_iters", C.c_int), ("halvings", C.c_int), ("status", C.c_int),
                ("res0", C.c_double), ("res", C.c_double), ("res_hist", C.c_double * 16), ("lin_hist", C.c_int * 16)]


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class tsp_allocator(C.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("ctx", C.c_void_p)]


class tsp_desc(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("rank", C.c_int), ("nranks", C.c_int),
                ("comm_kind", C.c_int), ("comm_arg", C.c_void_p),
                ("stream", C.c_void_p), ("inputs_on_device", C.c_int),
                ("A_uu", tsp_bsr), ("A_uf", tsp_bsr), ("A_fu", tsp_bsr), ("A_ff", tsp_bsr),
                ("fs_diag", C.c_void_p), ("opts", tsp_options), ("allocator", tsp_allocator)]


class TorchAllocator:
    """include/tsp.h tsp_allocator routed to torch's CUDA caching allocator
    (torch.cuda.caching_allocator_alloc / caching_allocator_delete): the library's device memory then lives in
    the same pool as the caller's tensors.  Marshalling only; counts the calls for the tests."""

    def __init__(self, torch, device):
        self.torch, self.device = torch, device
        self.allocs = self.frees = 0
        self.live_bytes = self.peak_bytes = 0

        def _alloc(nbytes, stream, ctx):
            try:
                p = torch.cuda.caching_allocator_alloc(int(nbytes), self.device, int(stream or 0))
            except Exception:                                   # out of memory: the library reports TSP_ERR_OOM
                return None
            self.allocs += 1
            self.live_bytes += int(nbytes)
            self.peak_bytes = max(self.peak_bytes, self.live_bytes)
            return p

        def _free(ptr, nbytes, stream, ctx):
            try:
                torch.cuda.caching_allocator_delete(ptr)
            except Exception:                                   # interpreter shutdown: torch is gone already
                return
            self.frees += 1
            self.live_bytes -= int(nbytes)

        self._cbs = (_ALLOC_FN(_alloc), _FREE_FN(_free))     # kept alive as long as the handle

    def struct(self):
        return tsp_allocator(self._cbs[0], self._cbs[1], None)


class tsp_solve_opts(C.Structure):
    _fields_ = [("rtol", C.c_double), ("restart", C.c_int), ("max_iters", C.c_int), ("x0_zero", C.c_int),
                ("host_ptrs", C.c_int)]


class tsp_solve_info(C.Structure):
    _fields_ = [("iterations", C.c_int), ("restarts", C.c_int), ("status", C.c_int),
                ("est_relres", C.c_double), ("true_relres", C.c_double), ("t_solve_s", C.c_double),
                ("reorth", C.c_int), ("bytes_krylov", C.c_double), ("dcgs_fallbacks", C.c_int)]


class tsp_stats(C.Structure):
    _fields_ = [("levels", C.c_int * 2), ("rows", (C.c_int64 * 16) * 2), ("nnz", (C.c_int64 * 16) * 2),
                ("launches", C.c_int64), ("skipped_dss", C.c_int64), ("perturbed_pivots", C.c_int64),
                ("coarsening_fallbacks", C.c_int64), ("bytes_apply", C.c_double), ("bytes_operator", C.c_double),
                ("bytes_iter_base", C.c_double), ("bytes_per_krylov_vec", C.c_double),
                ("allocs_callback", C.c_int64), ("allocs_pool", C.c_int64), ("bytes_live", C.c_int64)]


TSP_PROF_MAX = 32


class tsp_prof(C.Structure):
    _fields_ = [("nclasses", C.c_int), ("name", (C.c_char * 24) * TSP_PROF_MAX),
                ("launches", C.c_int64 * TSP_PROF_MAX), ("ms", C.c_double * TSP_PROF_MAX),
                ("bytes", C.c_double * TSP_PROF_MAX)]


def lib():
    """Load libtsp.so; raise loudly if it is missing (no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libtsp.so not built ({LIB_PATH}); run `make tsp` or __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.tsp_abi_version.restype = C.c_int
        L.tsp_last_error.restype = C.c_char_p
        L.tsp_default_options.argtypes = [_P(tsp_options)]
        L.tsp_create.argtypes = [_P(C.c_void_p), _P(tsp_desc)]
        L.tsp_setup.argtypes = [C.c_void_p, C.c_uint]
        L.tsp_update_values.argtypes = [C.c_void_p, _P(tsp_desc)]
        L.tsp_apply_preconditioner.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.tsp_apply_operator.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.tsp_solve.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, _P(tsp_solve_opts), _P(tsp_solve_info)]
        L.tsp_default_solve_opts.argtypes = [_P(tsp_solve_opts)]
        L.tsp_richardson.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, _P(tsp_solve_opts), _P(tsp_solve_info)]
        L.tsp_default_solve_opts.restype = None
        L.tsp_get_stats.argtypes = [C.c_void_p, _P(tsp_stats)]
        L.tsp_level_sizes.argtypes = [C.c_void_p, C.c_int, C.c_int, _P(C.c_int64)]
        L.tsp_export_level.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 8
        L.tsp_prof_enable.argtypes = [C.c_void_p, C.c_int]
        L.tsp_prof_classes.argtypes = [C.c_void_p, C.c_uint]
        L.tsp_export_cpr.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.tsp_prof_read.argtypes = [C.c_void_p, _P(tsp_prof)]
        L.tsp_destroy.argtypes = [C.c_void_p]
        L.tsp_destroy.restype = None
        L.tsp_nccl_unique_id.argtypes = [C.c_char_p]
        L.tsp_local_world_create.argtypes = [C.c_int]
        L.tsp_local_world_create.restype = C.c_void_p
        L.tsp_local_world_destroy.argtypes = [C.c_void_p]
        L.tsp_local_world_destroy.restype = None
        L.tsp_partition.argtypes = [C.c_int] * 6 + [_P(C.c_int64)]
        L.tsp_level_dist.argtypes = [C.c_void_p, C.c_int, C.c_int, _P(C.c_int64)]
        L.tsp_variant_counts.argtypes = [C.c_void_p, _P(C.c_int64)]
        L.tsp_export_colour.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, _P(C.c_int), _P(C.c_int)]
        L.tsp_assembly_sizes.argtypes = [_P(tsp_asm_params), C.c_int, C.c_int, C.c_int, _P(C.c_int64)]
        L.tsp_assemble.argtypes = [_P(tsp_asm_params), C.c_int, C.c_int, C.c_int, _P(tsp_cell_fields), _P(tsp_bsr_out),
                                   C.c_void_p, _P(C.c_double), C.c_void_p]
        L.tsp_assemble_scale.argtypes = [_P(tsp_asm_params), C.c_int, C.c_int, C.c_int, _P(C.c_double), _P(tsp_bsr_out),
                                         C.c_void_p, _P(C.c_double), C.c_void_p]
        L.tsp_residual.argtypes = [_P(tsp_asm_params), _P(tsp_cell_fields), C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p]
        L.tsp_masses.argtypes = [_P(tsp_asm_params), _P(tsp_cell_fields), C.c_void_p, C.c_void_p, C.c_void_p]
        L.tsp_newton_residual.argtypes = [C.c_void_p, _P(tsp_asm_params), _P(tsp_cell_fields), C.c_double, C.c_void_p,
                                          C.c_void_p, C.c_void_p]
        L.tsp_default_newton_opts.argtypes = [_P(tsp_newton_opts)]
        L.tsp_default_newton_opts.restype = None
        L.tsp_newton_step.argtypes = [C.c_void_p, _P(tsp_asm_params), _P(tsp_cell_fields), C.c_double, C.c_void_p, C.c_void_p,
                                      C.c_void_p, _P(tsp_newton_opts), _P(tsp_newton_info)]
        if L.tsp_abi_version() != 5:
            raise RuntimeError("libtsp ABI version mismatch")
        _LIB = L
    return _LIB


EXPORTED = ["tsp_abi_version", "tsp_last_error", "tsp_default_options", "tsp_create", "tsp_setup", "tsp_update_values",
            "tsp_apply_preconditioner", "tsp_apply_operator", "tsp_solve", "tsp_default_solve_opts", "tsp_richardson",
            "tsp_get_stats", "tsp_level_sizes", "tsp_export_level", "tsp_prof_enable", "tsp_prof_read",
            "tsp_prof_classes", "tsp_export_cpr", "tsp_destroy", "tsp_nccl_unique_id", "tsp_local_world_create", "tsp_local_world_destroy",
            "tsp_partition", "tsp_level_dist", "tsp_variant_counts", "tsp_export_colour",
            "tsp_assembly_sizes", "tsp_assemble", "tsp_assemble_scale", "tsp_residual", "tsp_masses",
            "tsp_default_newton_opts", "tsp_newton_step", "tsp_newton_residual"]

# include/tsp.h TSP_VAR_* order
VARIANTS = ["spgemm_hs64", "spgemm_hs128", "spgemm_hs512", "spgemm_hs4096", "spgemm_g4", "spgemm_g8", "spgemm_g32",
            "lanes_A0", "lanes_A8", "lanes_A16", "lanes_A32", "lanes_R0", "lanes_R8", "lanes_R16", "lanes_R32"]

TSP_COMM_NONE, TSP_COMM_NCCL, TSP_COMM_LOCAL = 0, 1, 2


def partition(nx, ny, nz, zblock, rank, nranks):
    """Owned ranges of a rank (include/tsp.h): k0, k1, first node, nodes, first cell, cells."""
    out = (C.c_int64 * 6)()
    _check(lib().tsp_partition(nx, ny, nz, zblock, rank, nranks, out), "tsp_partition")
    return tuple(out)


class AssembledProblem:
    """The blocks of tsp_assemble in device memory (torch CUDA tensors) with the attributes Tsp(...,
    device_inputs=True) reads; for a z-slab rank they are its owned rows with global column ids."""

    def __init__(self, nx, ny, nz, Nn, Nc, arrays, scales, row_max):
        self.nx, self.ny, self.nz, self.Nn, self.Nc = nx, ny, nz, Nn, Nc
        self.n = 3 * Nn + 2 * Nc
        self.scales, self.row_max = scales, row_max
        for k, v in arrays.items():
            setattr(self, k, v)


ASM_KEYS = ("nu", "biot", "gravity", "dt", "rho_w0", "rho_nw0", "c_w", "c_nw", "mu_w", "mu_nw", "rho_s", "p0",
            "swr", "snwr", "well_dbhp", "rw_over_h", "p_unit", "length", "burden", "dirichlet_bottom", "row_scale")


def assemble(params: dict, fields: dict, rank=0, nranks=1, zblock=16, stream=None, global_max=None):
    """GPU assembly of the Jacobian (tsp_assemble + tsp_assemble_scale).  `params`: the physical
    parameters (keys of include/tsp.h tsp_asm_params, e.g. synth.params_of(config)); `fields`: per-cell arrays of
    the GLOBAL grid (E, perm, phi, sat, pres as float64, well as int8; numpy or CUDA tensors).  `global_max`:
    callable turning this rank's 3 row maxima into the maxima over all ranks (needed when nranks > 1)."""
    import torch
    L = lib()
    P = tsp_asm_params(nx=params["nx"], ny=params["ny"], nz=params["nz"],
                       **{k: (int(params[k]) if k in ("burden", "dirichlet_bottom", "row_scale") else float(params[k]))
                          for k in ASM_KEYS})
    sz = (C.c_int64 * 6)()
    _check(L.tsp_assembly_sizes(C.byref(P), rank, nranks, zblock, sz), "tsp_assembly_sizes")
    Nn, Nc, Buu, Buf, Bfu, Bff = (int(v) for v in sz)
    dev = torch.device("cuda", torch.cuda.current_device())
    keep = {}
    for k in ("E", "perm", "phi", "sat", "pres"):
        keep[k] = torch.as_tensor(fields[k], dtype=torch.float64).to(dev).contiguous()
    if fields.get("well") is not None:
        keep["well"] = torch.as_tensor(fields["well"], dtype=torch.int8).to(dev).contiguous()
    if fields.get("phi0") is not None:
        keep["phi0"] = torch.as_tensor(fields["phi0"], dtype=torch.float64).to(dev).contiguous()
    f = tsp_cell_fields(*(keep[k].data_ptr() for k in ("E", "perm", "phi", "sat", "pres")),
                        keep["well"].data_ptr() if "well" in keep else None,
                        keep["phi0"].data_ptr() if "phi0" in keep else None)
    a = {}
    for name, rows, nb, bs in (("uu", Nn, Buu, 9), ("uf", Nn, Buf, 6), ("fu", Nc, Bfu, 6), ("ff", Nc, Bff, 4)):
        a[name + "_rowptr"] = torch.empty(rows + 1, dtype=torch.int32, device=dev)
        a[name + "_col"] = torch.empty(max(nb, 1), dtype=torch.int32, device=dev)
        a[name + "_val"] = torch.empty(max(nb, 1) * bs, dtype=torch.float64, device=dev)
    a["fs"] = torch.empty(max(2 * Nc, 1), dtype=torch.float64, device=dev)
    blocks = (tsp_bsr_out * 4)(*(tsp_bsr_out(a[n + "_rowptr"].data_ptr(), a[n + "_col"].data_ptr(), a[n + "_val"].data_ptr())
                                 for n in ("uu", "uf", "fu", "ff")))
    st = stream if stream is not None else torch.cuda.current_stream()
    rmax = (C.c_double * 3)()
    _check(L.tsp_assemble(C.byref(P), rank, nranks, zblock, C.byref(f), blocks, C.c_void_p(a["fs"].data_ptr()), rmax,
                          C.c_void_p(st.cuda_stream)), "tsp_assemble")
    mx = list(rmax)
    if nranks > 1:
        if global_max is None:
            raise ValueError("assemble: nranks > 1 needs global_max (the row maxima over all ranks)")
        mx = list(global_max(mx))
    gmx = (C.c_double * 3)(*mx)
    sc = (C.c_double * 3)()
    _check(L.tsp_assemble_scale(C.byref(P), rank, nranks, zblock, gmx, blocks, C.c_void_p(a["fs"].data_ptr()), sc,
                                C.c_void_p(st.cuda_stream)), "tsp_assemble_scale")
    return AssembledProblem(params["nx"], params["ny"], params["nz"], Nn, Nc, a, list(sc), mx)


def _asm_params(params):
    return tsp_asm_params(nx=params["nx"], ny=params["ny"], nz=params["nz"],
                          **{k: (int(params[k]) if k in ("burden", "dirichlet_bottom", "row_scale") else float(params[k]))
                             for k in ASM_KEYS})


def _ref_fields(ref):
    """tsp_cell_fields of the reference state: E, perm, phi (= phi_0), pres (= p_ref), well (CUDA tensors)."""
    return tsp_cell_fields(ref["E"].data_ptr(), ref["perm"].data_ptr(), ref["phi"].data_ptr(), None, ref["pres"].data_ptr(),
                           ref["well"].data_ptr() if ref.get("well") is not None else None, None)


def residual(params, ref, x, mprev, dt, out=None, stream=None):
    """tsp_residual: r(x) of Appendix B.1 in raw units (x = [u | (s, p [Pa])], CUDA tensors)."""
    import torch
    out = torch.empty_like(x) if out is None else out
    st = stream if stream is not None else torch.cuda.current_stream()
    P, f = _asm_params(params), _ref_fields(ref)
    _check(lib().tsp_residual(C.byref(P), C.byref(f), float(dt), C.c_void_p(x.data_ptr()), C.c_void_p(mprev.data_ptr()),
                              C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream)), "tsp_residual")
    return out


def masses(params, ref, x, stream=None):
    """tsp_masses: (V m_w, V m_nw) per cell at x."""
    import torch
    nc = params["nx"] * params["ny"] * params["nz"]
    m = torch.empty(2 * nc, dtype=torch.float64, device=x.device)
    st = stream if stream is not None else torch.cuda.current_stream()
    P, f = _asm_params(params), _ref_fields(ref)
    _check(lib().tsp_masses(C.byref(P), C.byref(f), C.c_void_p(x.data_ptr()), C.c_void_p(m.data_ptr()),
                            C.c_void_p(st.cuda_stream)), "tsp_masses")
    return m


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().tsp_nccl_unique_id(buf), "tsp_nccl_unique_id")
    return buf.raw


class LocalWorld:
    """Test backend: `n` ranks inside this process (one host thread per rank)."""

    def __init__(self, n):
        self.n = n
        self.h = lib().tsp_local_world_create(n)

    def close(self):
        if getattr(self, "h", None):
            lib().tsp_local_world_destroy(self.h)
            self.h = None

    __del__ = close


class TspError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = lib().tsp_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")


def _check(rc, where, ok=(0,)):
    if rc not in ok:
        raise TspError(rc, where)
    return rc


def _ptr(a):
    """Device pointer of a torch CUDA tensor, or host pointer of a numpy array."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        assert a.is_contiguous()
        return C.c_void_p(a.data_ptr())
    assert isinstance(a, np.ndarray) and a.flags["C_CONTIGUOUS"]
    return C.c_void_p(a.ctypes.data)


def default_options(**kw) -> tsp_options:
    o = tsp_options()
    lib().tsp_default_options(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


_LIVE = weakref.WeakSet()


@atexit.register
def _close_all():
    """Destroy the handles still open at exit while torch (whose allocator holds their memory) is alive."""
    for t in list(_LIVE):
        t.close()


class Tsp:
    """One handle.  `arrays` is a synth.Problem (numpy, host) -- or any object
    with the same attribute names holding CUDA torch tensors (device=True)."""

    def __init__(self, pb, stream=None, device_inputs=False, rank=0, nranks=1, comm_kind=0, comm_arg=None,
                 allocator="torch", **opts):
        """allocator: "torch" (default) routes every device buffer of the handle through torch's caching
        allocator (tsp_desc.allocator); None keeps the library's own stream-ordered pool."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libtsp needs a CUDA device (no CPU fallback)")
        L = lib()
        self.pb = pb
        self.n = pb.n
        self.torch = torch
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self._grid = (rank, nranks)
        keep = []
        d = self._desc(pb, device_inputs, keep)
        d.comm_kind = comm_kind
        if isinstance(comm_arg, (bytes, bytearray)):
            self._uid = C.create_string_buffer(bytes(comm_arg), 128)
            d.comm_arg = C.cast(self._uid, C.c_void_p)
        else:
            d.comm_arg = comm_arg
        d.stream = C.c_void_p(self.stream.cuda_stream)
        d.opts = default_options(**opts)
        self.allocator = None
        if allocator == "torch":
            self.allocator = TorchAllocator(torch, torch.cuda.current_device())
            d.allocator = self.allocator.struct()
        elif allocator is not None:
            raise ValueError("allocator must be 'torch' or None")
        h = C.c_void_p()
        _check(L.tsp_create(C.byref(h), C.byref(d)), "tsp_create")
        self.h = h
        _LIVE.add(self)

    def _desc(self, pb, device_inputs, keep):
        """tsp_desc with the grid, this rank and the four blocks + fs_diag of `pb` (arrays kept alive in `keep`)."""
        device_inputs = device_inputs or bool(getattr(pb.uu_val, "is_cuda", False))

        def arr(x):
            if device_inputs or hasattr(x, "data_ptr"):   # CUDA tensors, or pinned host tensors
                keep.append(x)
                return _ptr(x)
            y = np.ascontiguousarray(x)
            keep.append(y)
            return _ptr(y)

        d = tsp_desc()
        d.nx, d.ny, d.nz = pb.nx, pb.ny, pb.nz
        d.rank, d.nranks = self._grid
        d.inputs_on_device = int(device_inputs or bool(getattr(pb.uu_val, "is_cuda", False)))
        for name in ("uu", "uf", "fu", "ff"):
            b = tsp_bsr(arr(getattr(pb, name + "_rowptr")), arr(getattr(pb, name + "_col")), arr(getattr(pb, name + "_val")))
            setattr(d, "A_" + name, b)
        d.fs_diag = arr(pb.fs)
        return d

    def close(self):
        if getattr(self, "h", None):
            lib().tsp_destroy(self.h)
            self.h = None

    __del__ = close

    def setup(self, what=TSP_SETUP_MECH | TSP_SETUP_FLOW):
        _check(lib().tsp_setup(self.h, what), "tsp_setup")
        return self

    def update_values(self, pb, device_inputs=False):
        """tsp_update_values: a Newton step's new values on the same patterns (NEXT-f1)."""
        keep = []
        d = self._desc(pb, device_inputs, keep)
        _check(lib().tsp_update_values(self.h, C.byref(d)), "tsp_update_values")
        self.pb = pb
        return self

    def setup_flow(self, refresh=False):
        """tsp_setup(FLOW [| REFRESH]): the per-Newton flow phase; refresh keeps the pressure aggregation."""
        return self.setup(TSP_SETUP_FLOW | (TSP_SETUP_REFRESH if refresh else 0))

    def newton_residual(self, params, ref, x, dt, mprev=None, out=None):
        """tsp_newton_residual: this rank's residual rows at the rank-local state x (collective)."""
        out = self.torch.empty_like(x) if out is None else out
        P, f = _asm_params(params), _ref_fields(ref)
        _check(lib().tsp_newton_residual(self.h, C.byref(P), C.byref(f), float(dt), C.c_void_p(x.data_ptr()),
                                         C.c_void_p(mprev.data_ptr()) if mprev is not None else None,
                                         C.c_void_p(out.data_ptr())), "tsp_newton_residual")
        return out

    def newton_step(self, params, ref, x, mprev, dt, r_off=None, **opts):
        """tsp_newton_step: one implicit time step by Newton with line search (x updated in place; mprev None: the
        masses at x)."""
        o = tsp_newton_opts()
        lib().tsp_default_newton_opts(C.byref(o))
        for k, v in opts.items():
            setattr(o, k, v)
        info = tsp_newton_info()
        P, f = _asm_params(params), _ref_fields(ref)
        rc = lib().tsp_newton_step(self.h, C.byref(P), C.byref(f), float(dt), C.c_void_p(x.data_ptr()),
                                   C.c_void_p(mprev.data_ptr()) if mprev is not None else None,
                                   C.c_void_p(r_off.data_ptr()) if r_off is not None else None,
                                   C.byref(o), C.byref(info))
        _check(rc, "tsp_newton_step", ok=(0, 1))
        k = info.newton_iters
        return dict(newton_iters=k, lin_iters=info.lin_iters, halvings=info.halvings,
                    status="OK" if info.status == 0 else "NOT_CONVERGED", res0=info.res0, res=info.res,
                    res_hist=list(info.res_hist)[:min(k + 1, 16)], lin_hist=list(info.lin_hist)[:min(k, 16)])

    def apply_preconditioner(self, v, z):
        _check(lib().tsp_apply_preconditioner(self.h, _ptr(v), _ptr(z)), "tsp_apply_preconditioner")
        return z

    def apply_operator(self, x, y):
        _check(lib().tsp_apply_operator(self.h, _ptr(x), _ptr(y)), "tsp_apply_operator")
        return y

    def solve(self, b, x, rtol=1e-8, restart=64, max_iters=1000, x0_zero=True):
        """b, x: CUDA tensors (device) or numpy arrays (host; copies on the stream)."""
        host = isinstance(b, np.ndarray)
        o = tsp_solve_opts(rtol, restart, max_iters, int(x0_zero), int(host))
        info = tsp_solve_info()
        rc = lib().tsp_solve(self.h, _ptr(b), _ptr(x), C.byref(o), C.byref(info))
        _check(rc, "tsp_solve", ok=(0, 1))
        return dict(iterations=info.iterations, restarts=info.restarts, status=STATUS.get(info.status, info.status),
                    est_relres=info.est_relres, true_relres=info.true_relres, t_solve_s=info.t_solve_s,
                    reorth=info.reorth, bytes_krylov=info.bytes_krylov, dcgs_fallbacks=info.dcgs_fallbacks)

    def richardson(self, b, x, rtol=1e-8, max_iters=1000, x0_zero=True):
        """Sequential embedding x <- x + M^-1 (b - A x); arguments as solve()."""
        host = isinstance(b, np.ndarray)
        o = tsp_solve_opts(rtol, 1, max_iters, int(x0_zero), int(host))
        info = tsp_solve_info()
        rc = lib().tsp_richardson(self.h, _ptr(b), _ptr(x), C.byref(o), C.byref(info))
        _check(rc, "tsp_richardson", ok=(0, 1, -8))
        return dict(iterations=info.iterations, status=STATUS.get(info.status, info.status),
                    true_relres=info.true_relres, t_solve_s=info.t_solve_s)

    def stats(self):
        s = tsp_stats()
        _check(lib().tsp_get_stats(self.h, C.byref(s)), "tsp_get_stats")
        out = {f: getattr(s, f) for f, _ in tsp_stats._fields_ if f not in ("levels", "rows", "nnz")}
        out["levels"] = list(s.levels)
        out["rows"] = [list(s.rows[w])[: s.levels[w]] for w in range(2)]
        out["nnz"] = [list(s.nnz[w])[: s.levels[w]] for w in range(2)]
        return out

    def colour(self, which, lvl):
        """Test hook: (colour per row, gs_block, number of colours) of a level's Gauss-Seidel smoother."""
        n = self.level(which, lvl)["n"]
        col = np.empty(n, np.int32)
        blk, nc = C.c_int(0), C.c_int(0)
        _check(lib().tsp_export_colour(self.h, which, lvl, col.ctypes.data, C.byref(blk), C.byref(nc)), "tsp_export_colour")
        return col, blk.value, nc.value

    def variants(self):
        """Test hook: kernel-variant choices of this handle's setups (include/tsp.h tsp_variant_counts)."""
        o = (C.c_int64 * len(VARIANTS))()
        _check(lib().tsp_variant_counts(self.h, o), "tsp_variant_counts")
        return dict(zip(VARIANTS, list(o)))

    def num_levels(self, which):
        return self.stats()["levels"][which]

    def level(self, which, lvl):
        o = (C.c_int64 * 6)()
        _check(lib().tsp_level_sizes(self.h, which, lvl, o), "tsp_level_sizes")
        n, nnz, nagg, pnz, nc, coarsest = list(o)
        d = dict(n=n, nnz=nnz, nagg=nagg, nc=nc, coarsest=bool(coarsest))
        d["A_rp"] = np.empty(n + 1, np.int32); d["A_ci"] = np.empty(nnz, np.int32)
        d["A_v"] = np.empty((nnz, nc)); d["dl1"] = np.empty((n, nc))
        if not coarsest:
            d["agg"] = np.empty(n, np.int32); d["P_rp"] = np.empty(n + 1, np.int32)
            d["P_ci"] = np.empty(pnz, np.int32); d["P_v"] = np.empty((pnz, nc))
        _check(lib().tsp_export_level(self.h, which, lvl, *[_ptr(d.get(k)) for k in
                                      ("A_rp", "A_ci", "A_v", "agg", "P_rp", "P_ci", "P_v", "dl1")]), "tsp_export_level")
        return d

    def hierarchy(self, which):
        return [self.level(which, l) for l in range(self.num_levels(which))]

    def level_dist(self, which, lvl):
        o = (C.c_int64 * 3)()
        _check(lib().tsp_level_dist(self.h, which, lvl, o), "tsp_level_dist")
        return dict(dist=bool(o[0]), nglob=o[1], row_off=o[2])

    def prof_enable(self, on=True):
        _check(lib().tsp_prof_enable(self.h, int(on)), "tsp_prof_enable")

    def cpr(self):
        """Test hook: (D_ss^(CPR), D_ps^(CPR), D_fs used by a1 as (N_c, 2)) of this rank."""
        Nc = self.pb.Nc if not hasattr(self, "nc_local") else self.nc_local
        dss, dps, fs = np.empty(Nc), np.empty(Nc), np.empty(2 * Nc)
        _check(lib().tsp_export_cpr(self.h, dss.ctypes.data, dps.ctypes.data, fs.ctypes.data), "tsp_export_cpr")
        return dss, dps, fs.reshape(Nc, 2)

    def prof_classes(self, names=None):
        """Record only the named kernel classes (None: all)."""
        mask = 0xFFFFFFFF
        if names is not None:
            p = tsp_prof()
            _check(lib().tsp_prof_read(self.h, C.byref(p)), "tsp_prof_read")
            idx = {p.name[k].value.decode(): k for k in range(p.nclasses)}
            mask = 0
            for nm in names:
                mask |= 1 << idx[nm]
        _check(lib().tsp_prof_classes(self.h, mask), "tsp_prof_classes")

    def prof_read(self):
        p = tsp_prof()
        _check(lib().tsp_prof_read(self.h, C.byref(p)), "tsp_prof_read")
        return {p.name[k].value.decode(): dict(launches=p.launches[k], ms=p.ms[k], bytes=p.bytes[k])
                for k in range(p.nclasses) if p.launches[k]}
