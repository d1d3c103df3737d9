"""Thin ctypes binding of libpgcn.so (include/pgcn.h).  Argument marshalling only: every step of
the training path runs in the library's sm_100a kernels.  No CPU fallback: if the library is
missing or a call fails, this module raises.

Names follow the C ABI: `partition` (pgcn_partition, Alg. 1 l.1-5), `Context.layer_fwd`
(l.9-14), `Context.loss` (l.16), `Context.layer_bwd` (l.18-27), `Context.update` (l.31-32),
`Context.step` (one iteration t of Alg. 1).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PGCN_LIB") or os.path.join(HERE, "libpgcn.so")  # PGCN_LIB: dev A/B builds
MAX_LAYERS = 16
MAX_PARTS = 64

OK, EINVAL, ESTATE, ECUDA, ENCCL, ENOMEM, EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
T_H, T_HIN, T_Z, T_J, T_G = 0, 1, 2, 3, 4
XH_SKIP_F_WAIT, XH_SKIP_B_WAIT, XH_NOCOMM = 1, 2, 4  # pgcn_dev_exchange_hook flags (include/pgcn_dev.h)
KERNELS = ["spmm_fwd", "spmm_bwd", "gemm_fwd", "gemm_dw", "gemm_da", "dropout", "gather", "grad_reduce", "loss",
           "update", "spmm_tile_fwd", "spmm_tile_bwd"]


class PgcnError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("pgcn error %d: %s" % (code, msg))
        self.code = code


class PartView(C.Structure):
    _fields_ = [("part", C.c_int32), ("n_parts", C.c_int32), ("n_inner", C.c_int64), ("n_halo", C.c_int64),
                ("nnz", C.c_int64), ("n_send", C.c_int64),
                ("inner_gid", C.POINTER(C.c_int64)), ("halo_gid", C.POINTER(C.c_int64)),
                ("halo_off", C.POINTER(C.c_int64)), ("send_off", C.POINTER(C.c_int64)),
                ("send_idx", C.POINTER(C.c_int32)), ("row_ptr", C.POINTER(C.c_int64)),
                ("col_idx", C.POINTER(C.c_int32)), ("inv_deg", C.POINTER(C.c_float)),
                ("t_row_ptr", C.POINTER(C.c_int64)), ("t_col_idx", C.POINTER(C.c_int32)),
                ("inv_ptr", C.POINTER(C.c_int64)), ("inv_pos", C.POINTER(C.c_int32)),
                ("deg", C.POINTER(C.c_int64))]


class Config(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("width", C.c_int32 * (MAX_LAYERS + 1)), ("mode", C.c_int32),
                ("smooth_f", C.c_int32), ("smooth_g", C.c_int32), ("ema_init", C.c_int32),
                ("gamma", C.c_double), ("dropout", C.c_double), ("seed", C.c_uint64), ("gemm", C.c_int32),
                ("loss", C.c_int32), ("n_global", C.c_int64), ("n_train_global", C.c_int64), ("opt", C.c_int32),
                ("dump_j", C.c_int32), ("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("transform_first", C.c_int32), ("staleness_stats", C.c_int32),
                ("model", C.c_int32), ("depth", C.c_int32), ("gather", C.c_int32),
                ("train_sparse", C.c_int32), ("spmm_tiles", C.c_int32), ("tile_min", C.c_int32),
                ("transport", C.c_int32), ("halo_payload", C.c_int32), ("lean", C.c_int32)]


class Comm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("nccl_id_halo", C.c_void_p),
                ("nccl_id_reduce", C.c_void_p)]


class TensorDesc(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("rows", C.c_int64), ("cols", C.c_int64), ("ld", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libpgcn.so not built (%s): run `python -m paper_2203_10428_b200.build`" % LIB_PATH)
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
        L.pgcn_last_error.restype = C.c_char_p
        L.pgcn_partition.argtypes = [i64, vp, vp, i32, vp, i32, C.POINTER(vp)]
        L.pgcn_partition_view.argtypes = [vp, i32, C.POINTER(PartView)]
        L.pgcn_partition_n_nodes.argtypes = [vp]
        L.pgcn_partition_n_nodes.restype = i64
        L.pgcn_partition_free.argtypes = [vp]
        L.pgcn_partition_free.restype = None
        L.pgcn_workspace_bytes.argtypes = [vp, vp, i32, C.POINTER(Config), C.POINTER(C.c_size_t)]
        L.pgcn_ctx_create.argtypes = [vp, vp, i32, C.POINTER(Config), C.POINTER(Comm), vp, C.c_size_t, vp,
                                      C.POINTER(vp)]
        L.pgcn_ctx_destroy.argtypes = [vp]
        L.pgcn_set_inputs.argtypes = [vp, i32, vp, vp, vp]
        L.pgcn_stage_inputs.argtypes = [vp, i32, vp, i64, vp, vp]
        L.pgcn_param_count.argtypes = [C.POINTER(Config)]
        L.pgcn_param_count.restype = i64
        L.pgcn_layer_fwd.argtypes = [vp, i64, i32, vp]
        L.pgcn_loss.argtypes = [vp, i64, vp]
        L.pgcn_layer_bwd.argtypes = [vp, i64, i32, vp]
        L.pgcn_update.argtypes = [vp, i64, vp, vp, vp]
        L.pgcn_step.argtypes = [vp, i64, vp, vp, vp, vp]
        L.pgcn_layer_fwd_io.argtypes = [vp, i64, i32, vp, vp, vp, i64, vp, i64]
        L.pgcn_layer_bwd_io.argtypes = [vp, i64, i32, vp, vp, vp, i64, vp, vp, vp, i64]
        L.pgcn_tensor.argtypes = [vp, i32, i32, i32, i64, C.POINTER(TensorDesc)]
        L.pgcn_launch_count.argtypes = [vp]
        L.pgcn_launch_count.restype = i64
        L.pgcn_timing_enable.argtypes = [vp, i32]
        L.pgcn_timing_read_gather.argtypes = [vp, i32, C.POINTER(C.c_double)]
        L.pgcn_timing_read.argtypes = [vp, i32, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.pgcn_dev_gemm_scratch_bytes.argtypes = [i64, i64, i64]
        L.pgcn_dev_gemm_scratch_bytes.restype = C.c_size_t
        L.pgcn_dev_gemm.argtypes = [i32, i32, vp, vp, i64, i64, i64, vp, i64, vp, i64, vp, vp, i64, i32, vp,
                                    C.c_size_t, vp]
        L.pgcn_staleness.argtypes = [vp, i32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.pgcn_dev_spmm.argtypes = [vp, vp, vp, vp, i64, i64, i64, vp, vp]
        L.pgcn_dev_l2_read.argtypes = [vp, i64, i32, vp, vp]
        L.pgcn_dev_gather_read.argtypes = [vp, i64, vp, i64, vp, i32, vp]
        L.pgcn_dev_tiles.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp]
        L.pgcn_nccl_unique_id.argtypes = [vp]
        L.pgcn_dev_exchange_hook.argtypes = [vp, i64, i32]
        L.pgcn_dev_exchange_bytes.argtypes = [vp, vp, vp]
        L.pgcn_nccl_id_bytes.restype = i32
        L.pgcn_ipc_handle_bytes.restype = i32
        L.pgcn_ipc_export.argtypes = [vp, vp, C.POINTER(C.c_int64)]
        L.pgcn_ipc_import.argtypes = [vp, i32, vp, i64]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise PgcnError(rc, lib().pgcn_last_error().decode(errors="replace"))


def _ptr(a):
    """Address of a numpy array, torch tensor, or None."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


# ------------------------------------------------------------------------------------------- partition
class Partitioning:
    """pgcn_partition (Alg. 1 l.1-5) over a CSR graph."""

    def __init__(self, n, row_ptr, col_idx, n_parts, part_of=None, n_threads=0):
        # the CSR is borrowed for the duration of the call only (the handle owns copies of what it needs)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        col = np.ascontiguousarray(col_idx, dtype=np.int32)
        po = None if part_of is None else np.ascontiguousarray(part_of, dtype=np.int32)
        h = C.c_void_p()
        _check(lib().pgcn_partition(int(n), _ptr(rp), _ptr(col), int(n_parts), _ptr(po), int(n_threads), C.byref(h)))
        self.handle = h
        self.n = int(n)
        self.n_parts = int(n_parts)

    def raw_view(self, i) -> PartView:
        v = PartView()
        _check(lib().pgcn_partition_view(self.handle, int(i), C.byref(v)))
        return v

    def view(self, i) -> dict:
        """Copies of partition i's arrays (names of include/pgcn.h pgcn_part_view)."""
        v = self.raw_view(i)
        n_in, n_bd, nnz, ns, n_p = v.n_inner, v.n_halo, v.nnz, v.n_send, v.n_parts

        def arr(p, n, dt):
            if n == 0:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)
        return dict(part=v.part, n_parts=n_p, n_inner=n_in, n_halo=n_bd, nnz=nnz, n_send=ns,
                    inner_gid=arr(v.inner_gid, n_in, np.int64), halo_gid=arr(v.halo_gid, n_bd, np.int64),
                    halo_off=arr(v.halo_off, n_p + 1, np.int64), send_off=arr(v.send_off, n_p + 1, np.int64),
                    send_idx=arr(v.send_idx, ns, np.int32), row_ptr=arr(v.row_ptr, n_in + 1, np.int64),
                    col_idx=arr(v.col_idx, nnz, np.int32), inv_deg=arr(v.inv_deg, n_in, np.float32),
                    t_row_ptr=arr(v.t_row_ptr, n_in + n_bd + 1, np.int64), t_col_idx=arr(v.t_col_idx, nnz, np.int32),
                    inv_ptr=arr(v.inv_ptr, n_in + 1, np.int64), inv_pos=arr(v.inv_pos, ns, np.int32),
                    deg=arr(v.deg, n_in + n_bd, np.int64))

    def tiles(self, i, which, tile_min) -> dict:
        """pgcn_dev_tiles (include/pgcn_dev.h): the dense-tile decomposition of P_i (which = 0) or
        P_i^T (which = 1) used by the tensor-core aggregation."""
        sz = np.zeros(6, np.int64)
        _check(lib().pgcn_dev_tiles(self.handle, int(i), int(which), int(tile_min), _ptr(sz), None, None, None, None,
                                    None, None))
        n_rows, n_rb, n_tiles, nnz_heavy, nnz_light, n_cols = (int(x) for x in sz)
        out = dict(n_rows=n_rows, n_rb=n_rb, n_tiles=n_tiles, nnz_heavy=nnz_heavy, nnz_light=nnz_light, n_cols=n_cols,
                   rb_ptr=np.zeros(n_rb + 1, np.int32), order=np.zeros(n_rb, np.int32),
                   tile_col=np.zeros(n_tiles, np.int32), mask=np.zeros(128 * n_tiles, np.uint64),
                   lrp=np.zeros(n_rows + 1, np.int64), lcol=np.zeros(nnz_light, np.int32))
        _check(lib().pgcn_dev_tiles(self.handle, int(i), int(which), int(tile_min), _ptr(sz), _ptr(out["rb_ptr"]),
                                    _ptr(out["order"]), _ptr(out["tile_col"]), _ptr(out["mask"]), _ptr(out["lrp"]),
                                    _ptr(out["lcol"])))
        return out

    def close(self):
        if getattr(self, "handle", None):
            lib().pgcn_partition_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partition(n, row_ptr, col_idx, n_parts, part_of=None, n_threads=0) -> Partitioning:
    return Partitioning(n, row_ptr, col_idx, n_parts, part_of, n_threads)


# ------------------------------------------------------------------------------------------- config
def make_config(widths: Sequence[int], *, mode="pipe", smooth_f=False, smooth_g=False, gamma=0.95,
                ema_init="first", dropout=0.0, seed=4, gemm="tc", loss="ce", n_global=0, n_train_global=1,
                opt="adam", lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8, dump_j=False,
                transform_first=True, staleness_stats=False, model="sage", depth=1,
                gather="f32", train_sparse=False, spmm_tiles=True, tile_min=0, transport="local",
                halo_payload="f32", lean=False) -> Config:
    c = Config()
    c.n_layers = len(widths) - 1
    for i, w in enumerate(widths):
        c.width[i] = int(w)
    c.mode = {"vanilla": 0, "pipe": 1}[mode]
    c.smooth_f, c.smooth_g = int(bool(smooth_f)), int(bool(smooth_g))
    c.ema_init = {"first": 0, "zero": 1}[ema_init]
    c.gamma, c.dropout, c.seed = float(gamma), float(dropout), int(seed)
    c.gemm = {"tc": 0, "fp32": 0, "bf16": 1, "simt": 2}[gemm]
    c.loss = {"ce": 0, "bce": 1}[loss]
    c.n_global, c.n_train_global = int(n_global), int(n_train_global)
    c.opt = {"sgd": 0, "adam": 1}[opt]
    c.dump_j = int(bool(dump_j))
    c.lr, c.beta1, c.beta2, c.eps = float(lr), float(beta1), float(beta2), float(eps)
    c.transform_first = int(bool(transform_first))
    c.staleness_stats = int(bool(staleness_stats))
    c.model = {"sage": 0, "gcn": 1}[model]
    c.depth = int(depth)
    c.gather = {"f32": 0, "bf16": 1}[gather]
    c.train_sparse = int(bool(train_sparse))
    c.spmm_tiles = int(bool(spmm_tiles))
    c.tile_min = int(tile_min)
    c.transport = {"local": 0, "loopback": 1, "push": 2}[transport]
    c.halo_payload = {"f32": 0, "bf16": 1}[halo_payload]
    c.lean = int(bool(lean))
    return c


def workspace_bytes(part: "Partitioning", cfg: Config, local_parts: Optional[Sequence[int]] = None) -> int:
    """pgcn_workspace_bytes: device bytes a context hosting `local_parts` (default: all) needs."""
    loc = np.ascontiguousarray(list(range(part.n_parts)) if local_parts is None else local_parts, dtype=np.int32)
    nb = C.c_size_t()
    _check(lib().pgcn_workspace_bytes(part.handle, _ptr(loc), len(loc), C.byref(cfg), C.byref(nb)))
    return int(nb.value)


def param_count(cfg: Config) -> int:
    return int(lib().pgcn_param_count(C.byref(cfg)))


def flatten_params(layers) -> np.ndarray:
    """theta = vec[W^(1), b^(1), ..., W^(L), b^(L)] (include/pgcn.h layout), fp32."""
    return np.concatenate([np.concatenate([np.asarray(W, np.float32).ravel(), np.asarray(b, np.float32).ravel()])
                           for W, b in layers]).astype(np.float32)


def unflatten_params(theta, widths, model="sage"):
    out, o = [], 0
    k = 2 if model == "sage" else 1
    for fi, fo in zip(widths[:-1], widths[1:]):
        W = theta[o:o + k * fi * fo].reshape(k * fi, fo)
        o += k * fi * fo
        b = theta[o:o + fo]
        o += fo
        out.append((W, b))
    return out


# ------------------------------------------------------------------------------------------- NCCL bootstrap
def nccl_comm(rank: int, nranks: int, group=None) -> Comm:
    """pgcn_comm for a multi-process run: rank 0 draws two ncclUniqueIds (halo exchange and
    gradient all-reduce communicators) and torch.distributed broadcasts their bytes."""
    import torch
    import torch.distributed as dist
    nb = int(lib().pgcn_nccl_id_bytes())
    if nb <= 0:
        raise RuntimeError("libpgcn.so was built without NCCL")
    buf = np.zeros(2 * nb, dtype=np.uint8)
    if rank == 0:
        for k in range(2):
            tmp = (C.c_uint8 * nb)()
            _check(lib().pgcn_nccl_unique_id(C.addressof(tmp)))
            buf[k * nb:(k + 1) * nb] = np.frombuffer(bytes(tmp), dtype=np.uint8)
    t = torch.from_numpy(buf)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=0, group=group)
    ids = t.cpu().numpy().copy()
    cm = Comm()
    cm.rank, cm.nranks = int(rank), int(nranks)
    cm._ids = (C.c_uint8 * (2 * nb)).from_buffer_copy(ids.tobytes())
    cm.nccl_id_halo = C.addressof(cm._ids)
    cm.nccl_id_reduce = C.addressof(cm._ids) + nb
    return cm


# ------------------------------------------------------------------------------------------- context
class Context:
    """A pgcn_ctx hosting `local_parts` of a Partitioning on the current CUDA device."""

    def __init__(self, part: Partitioning, cfg: Config, local_parts: Optional[Sequence[int]] = None,
                 comm: Optional[Comm] = None, stream=None, device=None):
        import torch
        self.torch = torch
        self.part = part
        self.cfg = cfg
        self.local = np.ascontiguousarray(list(range(part.n_parts)) if local_parts is None else local_parts,
                                          dtype=np.int32)
        nb = C.c_size_t()
        _check(lib().pgcn_workspace_bytes(part.handle, _ptr(self.local), len(self.local), C.byref(cfg), C.byref(nb)))
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.ws = torch.empty(int(nb.value), dtype=torch.uint8, device=self.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        self._comm = comm
        _check(lib().pgcn_ctx_create(part.handle, _ptr(self.local), len(self.local), C.byref(cfg),
                                     C.byref(comm) if comm is not None else None, self.ws.data_ptr(),
                                     self.ws.numel(), self.stream.cuda_stream, C.byref(h)))
        self.handle = h
        self._keep = {}
        self.P = param_count(cfg)
        self.widths = [cfg.width[i] for i in range(cfg.n_layers + 1)]

    def ipc_connect(self, group=None):
        """N2 over NVLink (multi-process PUSH, include/pgcn.h pgcn_ipc_export): export this rank's workspace
        as a CUDA IPC handle, all-gather the handles with torch.distributed and map every peer's."""
        import torch.distributed as dist
        nb = int(lib().pgcn_ipc_handle_bytes())
        h = (C.c_uint8 * nb)()
        off = C.c_int64()
        _check(lib().pgcn_ipc_export(self.handle, C.addressof(h), C.byref(off)))
        rank = dist.get_rank(group)
        allh = [None] * dist.get_world_size(group)
        dist.all_gather_object(allh, (rank, bytes(h), int(off.value)), group=group)
        for r, hb, o in allh:
            if r == rank:
                continue
            buf = (C.c_uint8 * nb).from_buffer_copy(hb)
            _check(lib().pgcn_ipc_import(self.handle, int(r), C.addressof(buf), int(o)))
        dist.barrier(group)

    def set_inputs(self, local, X, labels, train_mask):
        """pgcn_set_inputs: the copies are asynchronous on the context stream, so the sources are kept
        alive per hosted partition until the next call for that partition (device tensors are also
        marked as used on the context stream for torch's caching allocator)."""
        srcs = (X, labels, train_mask)
        if any(getattr(a, "is_cuda", False) for a in srcs):
            # device inputs produced on the caller's current stream (e.g. a non_blocking H2D copy) must be
            # complete before the context stream reads them
            self.stream.wait_stream(self.torch.cuda.current_stream(self.device))
        for a in srcs:
            if hasattr(a, "record_stream") and getattr(a, "is_cuda", False):
                a.record_stream(self.stream)
        self._keep[int(local)] = srcs
        _check(lib().pgcn_set_inputs(self.handle, int(local), _ptr(X), _ptr(labels), _ptr(train_mask)))

    def stage_inputs(self, local, X, labels, train_mask):
        """pgcn_stage_inputs: per-iteration re-upload of partition `local`'s inputs from HOST memory
        (numpy arrays or pinned CPU tensors), overlapped with the iteration in flight.  X may be
        [n_inner x F_0] or already padded to [n_inner x round_up(F_0, 4)] (one contiguous copy)."""
        for a in (X, labels, train_mask):
            if getattr(a, "is_cuda", False):
                raise ValueError("stage_inputs takes host buffers")
        self._keep[("stage", int(local))] = (X, labels, train_mask)
        ld_x = int(X.stride(0)) if hasattr(X, "stride") and callable(X.stride) else int(X.strides[0] // 4)
        _check(lib().pgcn_stage_inputs(self.handle, int(local), _ptr(X), ld_x, _ptr(labels), _ptr(train_mask)))

    def layer_fwd(self, t, layer, params):
        _check(lib().pgcn_layer_fwd(self.handle, int(t), int(layer), _ptr(params)))

    @staticmethod
    def _ptr_array(tensors):
        """(ctypes void* array, row stride) of a per-hosted-partition list of 2-D tensors (None entries
        allowed), or (None, 0)."""
        if tensors is None:
            return None, 0
        arr = (C.c_void_p * len(tensors))(*[_ptr(x) for x in tensors])
        lds = {int(x.stride(0)) for x in tensors if x is not None}
        if len(lds) > 1:
            raise ValueError("all row strides must be equal")
        return arr, (lds.pop() if lds else 0)

    def layer_fwd_io(self, t, layer, W, b, h_in=None, h_out=None):
        """pgcn_layer_fwd_io: Alg. 1 l.9-14 with caller-owned W, b and per-partition H^(l-1) / H^(l)."""
        a_in, ld_in = self._ptr_array(h_in)
        a_out, ld_out = self._ptr_array(h_out)
        _check(lib().pgcn_layer_fwd_io(self.handle, int(t), int(layer), _ptr(W), _ptr(b), a_in, ld_in, a_out, ld_out))

    def layer_bwd_io(self, t, layer, W, b, j_out=None, dW_local=None, db_local=None, j_in=None):
        """pgcn_layer_bwd_io: Alg. 1 l.18-27 with caller-owned W, b, J^(l), G^(l) and J^(l-1)."""
        a_jo, ld_jo = self._ptr_array(j_out)
        a_ji, ld_ji = self._ptr_array(j_in)
        _check(lib().pgcn_layer_bwd_io(self.handle, int(t), int(layer), _ptr(W), _ptr(b), a_jo, ld_jo, _ptr(dW_local),
                                       _ptr(db_local), a_ji, ld_ji))

    def loss(self, t, loss_dev=None):
        _check(lib().pgcn_loss(self.handle, int(t), _ptr(loss_dev)))

    def layer_bwd(self, t, layer, params):
        _check(lib().pgcn_layer_bwd(self.handle, int(t), int(layer), _ptr(params)))

    def update(self, t, params, grads, opt_state=None):
        _check(lib().pgcn_update(self.handle, int(t), _ptr(params), _ptr(grads), _ptr(opt_state)))

    def step(self, t, params, grads, opt_state=None, loss_dev=None):
        _check(lib().pgcn_step(self.handle, int(t), _ptr(params), _ptr(grads), _ptr(opt_state), _ptr(loss_dev)))

    def tensor(self, local, kind, layer=0, t=1):
        """torch view (rows x cols, row stride ld) of an internal device buffer (pgcn_tensor)."""
        d = TensorDesc()
        _check(lib().pgcn_tensor(self.handle, int(local), int(kind), int(layer), int(t), C.byref(d)))
        torch = self.torch
        base = self.ws.data_ptr()
        off = (d.ptr - base)
        assert off % 4 == 0 and 0 <= off < self.ws.numel()
        f = self.ws.view(torch.float32) if self.ws.numel() % 4 == 0 else self.ws[: self.ws.numel() // 4 * 4].view(
            torch.float32)
        return torch.as_strided(f, (d.rows, d.cols), (d.ld, 1), off // 4)

    def timing_enable(self, on=True):
        _check(lib().pgcn_timing_enable(self.handle, int(bool(on))))

    def timing_read(self, kind):
        ms, n, by, fl = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        _check(lib().pgcn_timing_read(self.handle, int(kind), C.byref(ms), C.byref(n), C.byref(by), C.byref(fl)))
        gb = C.c_double()
        _check(lib().pgcn_timing_read_gather(self.handle, int(kind), C.byref(gb)))
        return dict(ms=ms.value, launches=n.value, bytes=by.value, flops=fl.value, gather_bytes=gb.value)

    def staleness(self, layer):
        """(feature error, gradient error) of the last iteration for `layer` (Fig. 5/7)."""
        f, g = C.c_double(), C.c_double()
        _check(lib().pgcn_staleness(self.handle, int(layer), C.byref(f), C.byref(g)))
        return f.value, g.value

    def exchange_hook(self, spin_ns=0, flags=0):
        """pgcn_dev_exchange_hook (include/pgcn_dev.h): delay / fault injection on the posted exchange."""
        _check(lib().pgcn_dev_exchange_hook(self.handle, int(spin_ns), int(flags)))

    def exchange_bytes(self):
        """pgcn_dev_exchange_bytes: (forward, backward) payload bytes posted so far."""
        f, b = C.c_int64(), C.c_int64()
        _check(lib().pgcn_dev_exchange_bytes(self.handle, C.byref(f), C.byref(b)))
        return f.value, b.value

    def launch_count(self) -> int:
        return int(lib().pgcn_launch_count(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            lib().pgcn_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------------------------------- diagnostics
def dev_gemm(op, variant, A0, A1, M, F, W_ext, N, out, ld_out, Mg=None, inv_deg=None, relu=False, stream=None):
    """pgcn_dev_gemm (include/pgcn_dev.h): one node-update GEMM on torch CUDA tensors."""
    import torch
    nb = int(lib().pgcn_dev_gemm_scratch_bytes(int(M), int(F), int(N)))
    scratch = torch.empty(max(nb, 256), dtype=torch.uint8, device=out.device)
    st = stream if stream is not None else torch.cuda.current_stream(out.device)
    ldA = A0.stride(0) if A0 is not None else 0
    ldM = Mg.stride(0) if Mg is not None else 0
    variant = {"tc": 0, "bf16": 1, "simt": 2}.get(variant, variant)
    _check(lib().pgcn_dev_gemm(int(op), int(variant), _ptr(A0), _ptr(A1), int(ldA), int(M), int(F), _ptr(W_ext),
                               int(N), _ptr(Mg), int(ldM), _ptr(inv_deg), _ptr(out), int(ld_out), int(bool(relu)),
                               scratch.data_ptr(), scratch.numel(), st.cuda_stream))
    return scratch
