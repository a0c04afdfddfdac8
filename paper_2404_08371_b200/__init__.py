"""paper_2404_08371_b200 -- B200-native matrix-free FE operator apply.

Python binding (ctypes) over the C ABI in include/tetmf_b200.h. The compute
path is the CUDA library ``_lib/libtetmf_b200.so`` (sm_100a); there is no CPU
fallback: importing this package without the built library raises.

Object model (mirrors the reference's FormSystem API, forms.hpp:41-89):
    ctx = Context("cube6", device=0)
    x = Function(ctx, SPACE_P1); y = Function(ctx, SPACE_P1)
    op = Operator(ctx, FORM_P1)
    x.fill_seeded(level, seed=42)
    op.apply(x, y, level)            # FormSystem::apply (Replace semantics)
    w = y.export_ref(level)          # reference global numbering
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TETMF_LIB") or os.path.join(_HERE, "_lib", "libtetmf_b200.so")

SPACE_P1, SPACE_P2, SPACE_ND1 = 0, 1, 2
FORM_P1, FORM_P2V, FORM_N1, FORM_P1K = 0, 1, 2, 3
REPLACE, ADD = 0, 1
COEFF_ALPHA, COEFF_BETA, COEFF_K, COEFF_CONST = 0, 1, 2, 3
FORM_SPACE = {FORM_P1: SPACE_P1, FORM_P1K: SPACE_P1, FORM_N1: SPACE_ND1, FORM_P2V: SPACE_P2}

EINVAL, EINTERNAL, EDEVICE, ECOMM = 1, 2, 3, 4
PARTITION_MACRO, PARTITION_SLAB = 0, 1
EXCHANGE_SENDRECV, EXCHANGE_PUT, EXCHANGE_PUT_PACK, EXCHANGE_PUT_FUSED = 0, 1, 2, 3


class TetmfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"tetmf error {code}: {msg}")
        self.code = code


class InvalidArgument(TetmfError, ValueError):
    pass


_lib: Optional[ctypes.CDLL] = None

_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_dp = ctypes.POINTER(ctypes.c_double)
_c_ip = ctypes.POINTER(ctypes.c_int)
_c_vp = ctypes.c_void_p

_SIGS = {
    "tetmf_last_error": (ctypes.c_char_p, []),
    "tetmf_version": (ctypes.c_char_p, []),
    "tetmf_ctx_create": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(_c_vp)]),
    "tetmf_ctx_create_dist": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_vp,
                                             ctypes.POINTER(_c_vp)]),
    "tetmf_ctx_destroy": (ctypes.c_int, [_c_vp]),
    "tetmf_ctx_create_mesh": (ctypes.c_int, [_c_dp, ctypes.c_int, _c_ip, ctypes.c_int, ctypes.c_int,
                                             ctypes.POINTER(_c_vp)]),
    "tetmf_loopback_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_c_vp)]),
    "tetmf_loopback_destroy": (ctypes.c_int, [_c_vp]),
    "tetmf_ctx_create_loopback": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, _c_vp, ctypes.c_int, ctypes.c_int,
                                                 ctypes.POINTER(_c_vp)]),
    "tetmf_ctx_create_dist_part": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_vp,
                                                  ctypes.c_int, ctypes.POINTER(_c_vp)]),
    "tetmf_ctx_transport_info": (ctypes.c_int, [_c_vp, ctypes.c_char_p, ctypes.c_int]),
    "tetmf_ctx_set_stream": (ctypes.c_int, [_c_vp, _c_vp]),
    "tetmf_ctx_synchronize": (ctypes.c_int, [_c_vp]),
    "tetmf_ctx_num_macros": (ctypes.c_int, [_c_vp, _c_ip, _c_ip]),
    "tetmf_ctx_local_macros": (ctypes.c_int, [_c_vp, _c_ip]),
    "tetmf_nccl_unique_id": (ctypes.c_int, [_c_vp]),
    "tetmf_fn_create": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.POINTER(_c_vp)]),
    "tetmf_fn_destroy": (ctypes.c_int, [_c_vp]),
    "tetmf_fn_size": (ctypes.c_int, [_c_vp, ctypes.c_int, _c_i64p]),
    "tetmf_fn_device_ptr": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.POINTER(_c_dp)]),
    "tetmf_fn_fill_seeded": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_int]),
    "tetmf_fn_fill_coefficient": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_double]),
    "tetmf_fn_upload": (ctypes.c_int, [_c_vp, ctypes.c_int, _c_dp, ctypes.c_int64]),
    "tetmf_fn_download": (ctypes.c_int, [_c_vp, ctypes.c_int, _c_dp, ctypes.c_int64]),
    "tetmf_fn_num_ref_dofs": (ctypes.c_int, [_c_vp, ctypes.c_int, _c_i64p]),
    "tetmf_fn_import_ref": (ctypes.c_int, [_c_vp, ctypes.c_int, _c_dp]),
    "tetmf_fn_export_ref": (ctypes.c_int, [_c_vp, ctypes.c_int, _c_dp]),
    "tetmf_fn_ref_owned_range": (ctypes.c_int, [_c_vp, ctypes.c_int, _c_i64p, _c_i64p]),
    "tetmf_fn_import_ref_owned": (ctypes.c_int, [_c_vp, ctypes.c_int, _c_dp]),
    "tetmf_fn_export_ref_owned": (ctypes.c_int, [_c_vp, ctypes.c_int, _c_dp]),
    "tetmf_op_create": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.POINTER(_c_vp), ctypes.c_int,
                                       ctypes.POINTER(_c_vp)]),
    "tetmf_op_destroy": (ctypes.c_int, [_c_vp]),
    "tetmf_apply": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, ctypes.c_int, ctypes.c_int]),
    "tetmf_apply_ref_host": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, ctypes.c_int, _c_dp, _c_dp]),
    "tetmf_apply_ref_host_batch": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, ctypes.c_int, ctypes.c_int,
                                                  ctypes.POINTER(_c_dp), ctypes.POINTER(_c_dp)]),
    "tetmf_host_alloc": (ctypes.c_int, [ctypes.POINTER(_c_vp), ctypes.c_int64]),
    "tetmf_host_free": (ctypes.c_int, [_c_vp]),
    "tetmf_plan_ref_map": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.c_int, _c_i64p, ctypes.c_int64, _c_i64p]),
    "tetmf_plan_layout": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.c_int, _c_i64p, _c_i64p]),
    "tetmf_plan_interior": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_ubyte),
                                           ctypes.c_int64]),
    "tetmf_plan_local_groups": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.c_int, _c_i64p, _c_i64p, _c_i64p,
                                               _c_i64p]),
    "tetmf_plan_exchange": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.c_int, _c_ip, _c_i64p, _c_i64p, _c_i64p,
                                           _c_i64p, _c_ip, _c_i64p, _c_i64p, _c_i64p, _c_i64p, _c_i64p]),
    "tetmf_host_local_sum": (ctypes.c_int, [_c_i64p, _c_i64p, ctypes.c_int64, _c_dp]),
    "tetmf_plan_slab_units": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_ip, _c_ip]),
    "tetmf_host_pack": (ctypes.c_int, [_c_dp, _c_i64p, ctypes.c_int64, _c_dp]),
    "tetmf_host_put_offsets": (ctypes.c_int, [ctypes.c_int, _c_i64p, ctypes.c_int, ctypes.c_int,
                                              ctypes.POINTER(ctypes.c_int), _c_i64p]),
    "tetmf_host_put_targets": (ctypes.c_int, [ctypes.c_int, _c_i64p, _c_i64p, _c_i64p,
                                              ctypes.POINTER(ctypes.c_int)]),
    "tetmf_selftest_nccl_put": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "tetmf_ctx_set_exchange_mode": (ctypes.c_int, [_c_vp, ctypes.c_int]),
    "tetmf_host_combine": (ctypes.c_int, [_c_dp, _c_dp, _c_i64p, _c_i64p, ctypes.c_int64]),
    "tetmf_measure_fp64_peak": (ctypes.c_int, [_c_vp, ctypes.c_double, _c_dp]),
    "tetmf_measure_fp64_peak2": (ctypes.c_int, [_c_vp, ctypes.c_double, _c_dp, _c_dp]),
    "tetmf_plan_local_matrix": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               _c_dp, _c_dp, _c_dp]),
    "tetmf_plan_stencil": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.c_int, _c_dp]),
    "tetmf_fn_dot": (ctypes.c_int, [_c_vp, _c_vp, ctypes.c_int, _c_dp]),
    "tetmf_fn_mask_dirichlet": (ctypes.c_int, [_c_vp, ctypes.c_int]),
    "tetmf_cg_solve": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, ctypes.c_int, ctypes.c_double, ctypes.c_int, _c_ip, _c_dp,
                                      _c_ip]),
    "tetmf_op_diagonal": (ctypes.c_int, [_c_vp, _c_vp, ctypes.c_int]),
    "tetmf_pcg_solve": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_vp, ctypes.c_int, ctypes.c_double, ctypes.c_int, _c_ip,
                                       _c_dp, _c_ip]),
    "tetmf_gradient": (ctypes.c_int, [_c_vp, _c_vp, ctypes.c_int]),
    "tetmf_gradient_transpose": (ctypes.c_int, [_c_vp, _c_vp, ctypes.c_int]),
    "tetmf_estimate_lambda_max": (ctypes.c_int, [_c_vp, _c_vp, ctypes.c_int, ctypes.c_int, _c_dp]),
    "tetmf_chebyshev_smooth": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                              ctypes.c_double]),
    "tetmf_op_profile": (ctypes.c_int, [_c_vp, ctypes.c_int]),
    "tetmf_op_set_variant": (ctypes.c_int, [_c_vp, ctypes.c_int]),
    "tetmf_op_set_quadrature": (ctypes.c_int, [_c_vp, ctypes.c_int]),
    "tetmf_op_kernel_stats": (ctypes.c_int, [_c_vp, _c_dp, _c_i64p]),
    "tetmf_op_debug_perturb_table": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.c_int64, ctypes.c_double]),
    "tetmf_launch_count": (ctypes.c_int, [_c_i64p]),
}


def slab_units(num_macros: int, level: int, nranks: int, rank: int) -> list[tuple[int, int, int]]:
    """(macro, za, zb) units of `rank` in the slab partition (planes za <= z < zb)."""
    n = ctypes.c_int()
    _check(lib().tetmf_plan_slab_units(num_macros, level, nranks, rank, ctypes.byref(n), None))
    buf = (ctypes.c_int * max(3 * n.value, 1))()
    _check(lib().tetmf_plan_slab_units(num_macros, level, nranks, rank, ctypes.byref(n), buf))
    return [tuple(buf[3 * i:3 * i + 3]) for i in range(n.value)]


def launch_count() -> int:
    n = ctypes.c_int64()
    _check(lib().tetmf_launch_count(ctypes.byref(n)))
    return n.value


def lib() -> ctypes.CDLL:
    """Loads the CUDA library; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"tetmf CUDA library missing: {LIB_PATH} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def _check(rc: int):
    if rc != 0:
        msg = lib().tetmf_last_error().decode()
        if rc == EINVAL:
            raise InvalidArgument(rc, msg)
        raise TetmfError(rc, msg)


def _dptr(a: np.ndarray, size: Optional[int] = None):
    """float64 C-contiguous array -> double*; size: required element count.
    Explicit checks (not asserts, which python -O strips): the C side copies
    exactly the count it expects, so a short array would overflow."""
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
        raise InvalidArgument(EINVAL, "expected a C-contiguous float64 numpy array")
    if size is not None and a.size != size:
        raise InvalidArgument(EINVAL, f"array has {a.size} entries, expected {size}")
    return a.ctypes.data_as(_c_dp)


def _iptr(a: np.ndarray, size: Optional[int] = None):
    if not isinstance(a, np.ndarray) or a.dtype != np.int64 or not a.flags.c_contiguous:
        raise InvalidArgument(EINVAL, "expected a C-contiguous int64 numpy array")
    if size is not None and a.size != size:
        raise InvalidArgument(EINVAL, f"array has {a.size} entries, expected {size}")
    return a.ctypes.data_as(_c_i64p)


class LoopbackGroup:
    """nranks virtual ranks of this process on one device (tetmf_loopback_*):
    the multi-rank apply's exchange and all-gather as device-to-device copies.
    Drive each rank's collective calls from its own thread (run_ranks)."""

    def __init__(self, nranks: int):
        h = _c_vp()
        _check(lib().tetmf_loopback_create(nranks, ctypes.byref(h)))
        self._h = h
        self.nranks = nranks

    @property
    def handle(self):
        return self._h

    def contexts(self, mesh: str, device: int = 0, partition: int = PARTITION_MACRO) -> list["Context"]:
        return [Context.loopback(self, mesh, r, device, partition) for r in range(self.nranks)]

    def close(self):
        if getattr(self, "_h", None):
            lib().tetmf_loopback_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_ranks(fn, nranks: int):
    """Runs fn(rank) for every rank in its own thread (ctypes releases the
    GIL during library calls, so the ranks meet at the collective steps);
    returns the results in rank order and re-raises the first failure."""
    import threading
    out, err = [None] * nranks, [None] * nranks

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out


class Context:
    """Mesh + topology + device + rank partition (FormSystem's inputs)."""

    def __init__(self, mesh: str, device: int = 0, rank: int = 0, nranks: int = 1,
                 nccl_id: Optional[bytes] = None, partition: int = PARTITION_MACRO):
        h = _c_vp()
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        _check(lib().tetmf_ctx_create_dist_part(mesh.encode(), device, rank, nranks,
                                                ctypes.cast(idbuf, _c_vp) if idbuf is not None else None,
                                                partition, ctypes.byref(h)))
        self._h = h
        self.mesh = mesh
        self.device = device
        self.rank = rank
        self.nranks = nranks

    @classmethod
    def from_arrays(cls, vertices, tets, device: int = 0, name: str = "in-memory") -> "Context":
        """Context over an in-memory macro mesh (tetmf_ctx_create_mesh):
        vertices (nv, 3) float64, tets (nt, 4) int vertex ids."""
        v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(tets, dtype=np.int32).reshape(-1, 4)
        self = cls.__new__(cls)
        h = _c_vp()
        _check(lib().tetmf_ctx_create_mesh(v.ctypes.data_as(_c_dp), v.shape[0], t.ctypes.data_as(_c_ip), t.shape[0],
                                           device, ctypes.byref(h)))
        self._h = h
        self.mesh, self.device, self.rank, self.nranks = name, device, 0, 1
        return self

    @classmethod
    def loopback(cls, group: "LoopbackGroup", mesh: str, rank: int, device: int = 0,
                 partition: int = PARTITION_MACRO) -> "Context":
        """Virtual rank `rank` of a loopback group (tetmf_ctx_create_loopback)."""
        self = cls.__new__(cls)
        h = _c_vp()
        _check(lib().tetmf_ctx_create_loopback(mesh.encode(), device, group.handle, rank, partition,
                                               ctypes.byref(h)))
        self._h = h
        self.mesh, self.device, self.rank, self.nranks = mesh, device, rank, group.nranks
        self._group = group  # keeps the group alive as long as its contexts
        return self

    def transport_info(self) -> str:
        buf = ctypes.create_string_buffer(256)
        _check(lib().tetmf_ctx_transport_info(self._h, buf, 256))
        return buf.value.decode()

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().tetmf_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_exchange_mode(self, mode: int):
        """EXCHANGE_SENDRECV (default), EXCHANGE_PUT (slab partition: the P1
        stencil kernel issues its puts itself; else the pack kernel),
        EXCHANGE_PUT_PACK (always the pack kernel) or EXCHANGE_PUT_FUSED
        (always in-kernel for P1); before the first level is used."""
        _check(lib().tetmf_ctx_set_exchange_mode(self._h, int(mode)))

    def set_stream(self, stream_ptr: int):
        _check(lib().tetmf_ctx_set_stream(self._h, _c_vp(stream_ptr)))

    def synchronize(self):
        _check(lib().tetmf_ctx_synchronize(self._h))

    def num_macros(self):
        g, l = ctypes.c_int(), ctypes.c_int()
        _check(lib().tetmf_ctx_num_macros(self._h, ctypes.byref(g), ctypes.byref(l)))
        return g.value, l.value

    def local_macros(self):
        _, l = self.num_macros()
        out = (ctypes.c_int * max(l, 1))()
        _check(lib().tetmf_ctx_local_macros(self._h, out))
        return list(out)[:l]

    # ---- planning hooks (no GPU needed)
    def layout(self, space: int, level: int):
        ms, cs = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().tetmf_plan_layout(self._h, space, level, ctypes.byref(ms), ctypes.byref(cs)))
        return ms.value, cs.value

    def ref_map(self, space: int, level: int) -> tuple[np.ndarray, int]:
        ms, _ = self.layout(space, level)
        total = ms * len(self.local_macros())
        out = np.empty(total, dtype=np.int64)
        nd = ctypes.c_int64()
        _check(lib().tetmf_plan_ref_map(self._h, space, level, _iptr(out), total, ctypes.byref(nd)))
        return out, nd.value

    def interior(self, space: int, level: int) -> np.ndarray:
        """Interior (non-Dirichlet) mask in reference numbering (uint8)."""
        _, nd = self.ref_map(space, level)
        out = np.empty(nd, dtype=np.uint8)
        _check(lib().tetmf_plan_interior(self._h, space, level, out.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte)), nd))
        return out

    def local_groups(self, space: int, level: int):
        ng, nc = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().tetmf_plan_local_groups(self._h, space, level, ctypes.byref(ng), ctypes.byref(nc), None, None))
        off = np.empty(ng.value + 1, dtype=np.int64)
        cp = np.empty(max(nc.value, 1), dtype=np.int64)
        _check(lib().tetmf_plan_local_groups(self._h, space, level, None, None, _iptr(off), _iptr(cp)))
        return off, cp[: nc.value]

    def exchange_plan(self, space: int, level: int) -> dict:
        npeers = ctypes.c_int()
        ns, nr, ng, ne = (ctypes.c_int64() for _ in range(4))
        L = lib()
        _check(L.tetmf_plan_exchange(self._h, space, level, ctypes.byref(npeers), ctypes.byref(ns), ctypes.byref(nr),
                                     ctypes.byref(ng), ctypes.byref(ne), None, None, None, None, None, None))
        peers = (ctypes.c_int * max(npeers.value, 1))()
        so = np.empty(npeers.value + 1, dtype=np.int64)
        ro = np.empty(npeers.value + 1, dtype=np.int64)
        si = np.empty(max(ns.value, 1), dtype=np.int64)
        go = np.empty(ng.value + 1, dtype=np.int64)
        ge = np.empty(max(ne.value, 1), dtype=np.int64)
        _check(L.tetmf_plan_exchange(self._h, space, level, None, None, None, None, None, peers, _iptr(so),
                                     _iptr(ro), _iptr(si), _iptr(go), _iptr(ge)))
        return {"peers": list(peers)[: npeers.value], "send_offsets": so, "recv_offsets": ro,
                "send_index": si[: ns.value], "group_offsets": go, "group_entries": ge[: ne.value]}

    def local_matrix(self, form: int, level: int, macro: int, orientation: int, c0=None, c1=None) -> np.ndarray:
        nloc = 6 if form == FORM_N1 else (10 if form == FORM_P2V else 4)
        out = np.empty(nloc * nloc)
        a = None if c0 is None else np.ascontiguousarray(c0, dtype=np.float64)
        b = None if c1 is None else np.ascontiguousarray(c1, dtype=np.float64)
        _check(lib().tetmf_plan_local_matrix(self._h, form, level, macro, orientation,
                                             _dptr(a) if a is not None else None,
                                             _dptr(b) if b is not None else None, _dptr(out)))
        return out.reshape(nloc, nloc)

    def stencil(self, level: int, macro: int) -> np.ndarray:
        out = np.empty(16 * 15)
        _check(lib().tetmf_plan_stencil(self._h, level, macro, _dptr(out)))
        return out.reshape(16, 15)

    def fp64_peak(self, seconds: float = 1.0) -> float:
        tf = ctypes.c_double()
        _check(lib().tetmf_measure_fp64_peak(self._h, seconds, ctypes.byref(tf)))
        return tf.value

    def fp64_peak2(self, seconds: float = 4.0) -> tuple[float, float]:
        """(burst, sustained) FP64 TFLOP/s of the DFMA-chain probe."""
        b, s = ctypes.c_double(), ctypes.c_double()
        _check(lib().tetmf_measure_fp64_peak2(self._h, seconds, ctypes.byref(b), ctypes.byref(s)))
        return b.value, s.value


class Function:
    """Level-indexed per-macro lattice storage of one space (device)."""

    def __init__(self, ctx: Context, space: int):
        h = _c_vp()
        _check(lib().tetmf_fn_create(ctx.handle, space, ctypes.byref(h)))
        self._h = h
        self.ctx = ctx
        self.space = space

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().tetmf_fn_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def size(self, level: int) -> int:
        n = ctypes.c_int64()
        _check(lib().tetmf_fn_size(self._h, level, ctypes.byref(n)))
        return n.value

    def device_ptr(self, level: int) -> int:
        p = _c_dp()
        _check(lib().tetmf_fn_device_ptr(self._h, level, ctypes.byref(p)))
        return ctypes.cast(p, _c_vp).value

    def fill_seeded(self, level: int, seed: int, dirichlet_zero: bool = False):
        _check(lib().tetmf_fn_fill_seeded(self._h, level, seed, int(dirichlet_zero)))

    def fill_coefficient(self, level: int, which: int, value: float = 0.0):
        _check(lib().tetmf_fn_fill_coefficient(self._h, level, which, value))

    def upload(self, level: int, data: np.ndarray):
        data = np.ascontiguousarray(data, dtype=np.float64)
        _check(lib().tetmf_fn_upload(self._h, level, _dptr(data), data.size))

    def download(self, level: int) -> np.ndarray:
        out = np.empty(self.size(level), dtype=np.float64)
        _check(lib().tetmf_fn_download(self._h, level, _dptr(out), out.size))
        return out

    def num_ref_dofs(self, level: int) -> int:
        n = ctypes.c_int64()
        _check(lib().tetmf_fn_num_ref_dofs(self._h, level, ctypes.byref(n)))
        return n.value

    def import_ref(self, level: int, v: np.ndarray):
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.size != self.num_ref_dofs(level):
            raise InvalidArgument(EINVAL, "import_ref: vector length does not match num_ref_dofs")
        _check(lib().tetmf_fn_import_ref(self._h, level, _dptr(v)))

    def export_ref(self, level: int) -> np.ndarray:
        out = np.empty(self.num_ref_dofs(level), dtype=np.float64)
        _check(lib().tetmf_fn_export_ref(self._h, level, _dptr(out)))
        return out

    def owned_ref_range(self, level: int) -> tuple[int, int]:
        """[lo, hi): this rank's owned slice of the reference numbering."""
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().tetmf_fn_ref_owned_range(self._h, level, ctypes.byref(lo), ctypes.byref(hi)))
        return lo.value, hi.value

    def import_ref_owned(self, level: int, v):
        """Owned slice in (numpy array of hi - lo entries, or a raw pinned host
        pointer), ghost copies from their owners (collective)."""
        lo, hi = self.owned_ref_range(level)
        p = _dptr(v, hi - lo) if isinstance(v, np.ndarray) else ctypes.cast(_c_vp(v), _c_dp)
        _check(lib().tetmf_fn_import_ref_owned(self._h, level, p))

    def export_ref_owned(self, level: int, out=None):
        lo, hi = self.owned_ref_range(level)
        if out is None:
            out = np.empty(hi - lo)
        p = _dptr(out, hi - lo) if isinstance(out, np.ndarray) else ctypes.cast(_c_vp(out), _c_dp)
        _check(lib().tetmf_fn_export_ref_owned(self._h, level, p))
        return out

    def dot(self, other: "Function", level: int) -> float:
        """Inner product over the interior (non-Dirichlet) carriers, each once."""
        out = ctypes.c_double()
        _check(lib().tetmf_fn_dot(self._h, other.handle, level, ctypes.byref(out)))
        return out.value

    def mask_dirichlet(self, level: int):
        """Zero the Dirichlet (domain-boundary) carriers."""
        _check(lib().tetmf_fn_mask_dirichlet(self._h, level))


class Operator:
    """Form + coefficient functions (FormSystem + coefficient binding)."""

    def __init__(self, ctx: Context, form: int, coeffs: Sequence[Function] = ()):
        arr = (_c_vp * max(len(coeffs), 1))(*[c.handle for c in coeffs])
        h = _c_vp()
        _check(lib().tetmf_op_create(ctx.handle, form, arr, len(coeffs), ctypes.byref(h)))
        self._h = h
        self.ctx = ctx
        self.form = form
        self._coeffs = list(coeffs)  # keep alive (borrowed by the library)

    def close(self):
        if getattr(self, "_h", None):
            lib().tetmf_op_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def apply(self, src: Function, dst: Function, level: int, update: int = REPLACE):
        _check(lib().tetmf_apply(self._h, src.handle, dst.handle, level, update))

    def apply_ref_host(self, src: Function, dst: Function, level: int, v, w):
        """v, w: float64 numpy arrays of num_ref_dofs(level) entries (checked)
        or raw (pinned) host pointers (int) of that many doubles."""
        nd = src.num_ref_dofs(level)
        pv = _dptr(v, nd) if isinstance(v, np.ndarray) else ctypes.cast(_c_vp(v), _c_dp)
        pw = _dptr(w, nd) if isinstance(w, np.ndarray) else ctypes.cast(_c_vp(w), _c_dp)
        _check(lib().tetmf_apply_ref_host(self._h, src.handle, dst.handle, level, pv, pw))

    def apply_ref_host_batch(self, src: Function, dst: Function, level: int, vs, ws):
        """w_k = A v_k for lists of float64 numpy arrays or raw (pinned) host
        pointers (int), pipelined (tetmf_apply_ref_host_batch)."""
        if len(vs) != len(ws):
            raise InvalidArgument(EINVAL, "apply_ref_host_batch: len(vs) != len(ws)")
        nd = src.num_ref_dofs(level)

        def ptr(a):
            return _dptr(a, nd) if isinstance(a, np.ndarray) else ctypes.cast(_c_vp(a), _c_dp)
        pv = (_c_dp * len(vs))(*[ptr(a) for a in vs])
        pw = (_c_dp * len(ws))(*[ptr(a) for a in ws])
        _check(lib().tetmf_apply_ref_host_batch(self._h, src.handle, dst.handle, level, len(vs), pv, pw))

    def cg_solve(self, b: Function, x: Function, level: int, rtol: float = 1e-10, max_iter: int = 1000,
                 diag: Function | None = None):
        """Dirichlet-masked CG for A x = b (x: initial guess in, solution out);
        diag (from diagonal()) -> Jacobi-preconditioned CG.
        Returns (iterations, relative residual, converged)."""
        it = ctypes.c_int()
        rr = ctypes.c_double()
        cv = ctypes.c_int()
        if diag is None:
            _check(lib().tetmf_cg_solve(self._h, b.handle, x.handle, level, rtol, max_iter, ctypes.byref(it),
                                        ctypes.byref(rr), ctypes.byref(cv)))
        else:
            _check(lib().tetmf_pcg_solve(self._h, b.handle, x.handle, diag.handle, level, rtol, max_iter,
                                         ctypes.byref(it), ctypes.byref(rr), ctypes.byref(cv)))
        return it.value, rr.value, bool(cv.value)

    def lambda_max(self, diag: Function, level: int, iterations: int = 30) -> float:
        """Largest eigenvalue of D^-1 A (power iteration)."""
        out = ctypes.c_double()
        _check(lib().tetmf_estimate_lambda_max(self._h, diag.handle, level, iterations, ctypes.byref(out)))
        return out.value

    def chebyshev_smooth(self, diag: Function, b: Function, x: Function, level: int, degree: int,
                         lambda_max: float, eig_ratio: float = 30.0):
        """degree Chebyshev-Jacobi steps towards A x = b (x updated in place)."""
        _check(lib().tetmf_chebyshev_smooth(self._h, diag.handle, b.handle, x.handle, level, degree, lambda_max,
                                            eig_ratio))

    def debug_perturb_table(self, level: int, index: int, delta: float):
        """Negative-control hook: corrupts one table entry the kernel reads."""
        _check(lib().tetmf_op_debug_perturb_table(self._h, level, index, delta))

    def diagonal(self, d: Function, level: int):
        """d = diag(A) (the assembled operator's diagonal; all copies hold the sum)."""
        _check(lib().tetmf_op_diagonal(self._h, d.handle, level))

    def set_variant(self, variant: int):
        """0 = optimized kernels (default), 1 = first-version kernels."""
        _check(lib().tetmf_op_set_variant(self._h, variant))

    def set_quadrature(self, degree: int):
        """0 = exact integration (default), 1..6 = the reference's
        quadrature(degree) (FormSystem::apply(v, coeffs, quadrature(d)))."""
        _check(lib().tetmf_op_set_quadrature(self._h, degree))

    def profile(self, enable: bool = True):
        _check(lib().tetmf_op_profile(self._h, int(enable)))

    def kernel_stats(self):
        ms = ctypes.c_double()
        n = ctypes.c_int64()
        _check(lib().tetmf_op_kernel_stats(self._h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value


def gradient(p1: Function, nd1: Function, level: int):
    """nd1 = G p1: (G p)_e = p(tip) - p(base) (ND1 interpolant of grad p)."""
    _check(lib().tetmf_gradient(p1.handle, nd1.handle, level))


def gradient_transpose(nd1: Function, p1: Function, level: int):
    """p1 = G^T nd1."""
    _check(lib().tetmf_gradient_transpose(nd1.handle, p1.handle, level))


def host_local_sum(offsets, copies, y):
    _check(lib().tetmf_host_local_sum(_iptr(offsets), _iptr(copies), offsets.size - 1, _dptr(y)))


def host_put_offsets(counts, rank, peers):
    """where `rank`'s values start in each peer's receive buffer (counts[src, dst])"""
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    peers = np.ascontiguousarray(peers, dtype=np.int32)
    out = np.zeros(max(peers.size, 1), dtype=np.int64)
    _check(lib().tetmf_host_put_offsets(counts.shape[0], _iptr(counts), int(rank), peers.size,
                                        peers.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), _iptr(out)))
    return out[:peers.size]


def host_put_targets(send_offsets, peer_off):
    """per send entry: (position in the target peer's receive buffer, peer slot)"""
    send_offsets = np.ascontiguousarray(send_offsets, dtype=np.int64)
    peer_off = np.ascontiguousarray(peer_off, dtype=np.int64)
    n = int(send_offsets[-1])
    dst = np.zeros(max(n, 1), dtype=np.int64)
    slot = np.zeros(max(n, 1), dtype=np.int32)
    _check(lib().tetmf_host_put_targets(send_offsets.size - 1, _iptr(send_offsets),
                                        _iptr(peer_off if peer_off.size else np.zeros(1, np.int64)),
                                        _iptr(dst), slot.ctypes.data_as(ctypes.POINTER(ctypes.c_int))))
    return dst[:n], slot[:n]


def selftest_nccl_put(device=0, rounds=4):
    _check(lib().tetmf_selftest_nccl_put(int(device), int(rounds)))


def host_pack(y, send_index):
    out = np.empty(send_index.size, dtype=np.float64)
    if send_index.size:
        _check(lib().tetmf_host_pack(_dptr(y), _iptr(send_index), send_index.size, _dptr(out)))
    return out


def host_combine(y, recv, group_offsets, group_entries):
    recv = np.ascontiguousarray(recv, dtype=np.float64)
    if recv.size == 0:
        recv = np.zeros(1)
    _check(lib().tetmf_host_combine(_dptr(y), _dptr(recv), _iptr(group_offsets), _iptr(group_entries),
                                    group_offsets.size - 1))


def host_alloc(nbytes: int) -> int:
    p = _c_vp()
    _check(lib().tetmf_host_alloc(ctypes.byref(p), nbytes))
    return p.value


def host_free(ptr: int):
    _check(lib().tetmf_host_free(_c_vp(ptr)))


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().tetmf_nccl_unique_id(buf))
    return buf.raw
