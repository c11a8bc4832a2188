"""Thin Python binding of libfhash.so (include/fhash.h) -- argument
marshalling only.  Every step of the path runs in the library's sm_100a
kernels; there is NO CPU fallback: if the shared library is missing or a
call fails, this module raises.

Torch is used for device memory and streams only: tensors are passed to the
C ABI as raw device pointers on the current CUDA stream.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FHASH_LIB", os.path.join(_PKG, "libfhash.so"))  # override: experiments only

FH_OK, FH_E_ARG, FH_E_RANGE, FH_E_DOMAIN, FH_E_CUDA, FH_E_DIVERGED, FH_E_STATE = 0, -1, -2, -3, -4, -5, -6
FH_F32, FH_F16, FH_BF16 = 0, 1, 2
MAX_LEVELS = 32

_STATUS_NAMES = {0: "FH_OK", -1: "FH_E_ARG", -2: "FH_E_RANGE", -3: "FH_E_DOMAIN", -4: "FH_E_CUDA",
                 -5: "FH_E_DIVERGED", -6: "FH_E_STATE"}

# Every symbol include/fhash.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "fh_fold_schedule", "fh_build_levels", "fh_level_info_get", "fh_num_levels", "fh_feature_dim",
    "fh_table_entries", "fh_param_count", "fh_encoder_destroy", "fh_encode_fwd", "fh_encode_bwd", "fh_encode_bwd_ex",
    "fh_encode_indices", "fh_zero_grad", "fh_encode_fwd_bwd", "fh_encode_step_host", "fh_status_sync", "fh_last_error",
    "fh_version", "fh_build_mhe", "fh_encoder_kind", "fh_build_levels_lin",
    # include/fhash_bench.h (measurement kernels)
    "fh_bench_gather", "fh_bench_red", "fh_bench_copy", "fh_bench_gather_levels", "fh_bench_red_levels",
    # train step
    "fh_mlp_param_count", "fh_train_workspace_size", "fh_trainer_create", "fh_train_fwd_bwd", "fh_train_apply",
    "fh_train_step", "fh_trainer_status", "fh_trainer_step_count", "fh_trainer_destroy", "fh_train_apply_sharded",
    "fh_train_dx_layout", "fh_train_bwd_launches", "fh_train_bwd_ranges", "fh_train_set_bwd_events", "fh_train_apply_ranges",
    "fh_train_apply_peers", "fh_train_apply_multicast", "fh_nccl_unique_id", "fh_nccl_comm_create", "fh_nccl_comm_destroy",
    "fh_trainer_dp_workspace_size", "fh_trainer_set_comm", "fh_level_stats_workspace_size", "fh_level_stats", "fh_kernel_launches", "fh_encoder_scratch_size", "fh_encoder_attach_scratch",
    # inference (renderer's model evaluation) and the ARM pace rule
    "fh_infer_workspace_size", "fh_infer", "fh_arm_pace",
    # include/fhash_coreset.h (NEXT-4 coreset selection)
    "fh_coreset_workspace_size", "fh_occupancy_words", "fh_morton_cell", "fh_coreset_build", "fh_coreset_emit",
    # include/fhash_data.h (synthetic data, harness)
    "fh_data_gaussian_blobs", "fh_data_value_noise", "fh_data_normalize", "fh_data_sample_voxels",
]


class FHashError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class LevelRes(ctypes.Structure):
    _fields_ = [("res", ctypes.c_uint32 * 4)]


class LevelInfo(ctypes.Structure):
    _fields_ = [("res", ctypes.c_uint32 * 4), ("corners", ctypes.c_uint64), ("table_size", ctypes.c_uint64),
                ("hashed", ctypes.c_uint32), ("lin", ctypes.c_uint32), ("offset", ctypes.c_uint64)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load the in-tree libfhash.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, u64, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
    L.fh_fold_schedule.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.POINTER(LevelRes), ctypes.POINTER(c_int)]
    L.fh_build_levels.argtypes = [ctypes.POINTER(LevelRes), c_int, c_int, c_int, u64, ctypes.POINTER(vp)]
    L.fh_build_levels_lin.argtypes = [ctypes.POINTER(LevelRes), c_int, c_int, c_int, u64, c_int, ctypes.POINTER(vp)]
    L.fh_build_levels_lin.restype = c_int
    L.fh_level_info_get.argtypes = [vp, c_int, ctypes.POINTER(LevelInfo)]
    L.fh_num_levels.argtypes = [vp]
    L.fh_feature_dim.argtypes = [vp]
    L.fh_table_entries.argtypes = [vp]
    L.fh_table_entries.restype = u64
    L.fh_param_count.argtypes = [vp]
    L.fh_param_count.restype = u64
    L.fh_encoder_destroy.argtypes = [vp]
    L.fh_encoder_destroy.restype = None
    L.fh_encode_fwd.argtypes = [vp, vp, i64, vp, vp, c_int, vp]
    L.fh_encode_bwd.argtypes = [vp, vp, i64, vp, vp, vp]
    L.fh_encode_indices.argtypes = [vp, vp, i64, vp, vp, vp]
    L.fh_encode_fwd_bwd.argtypes = [vp, vp, i64, vp, vp, c_int, vp, vp, c_int, vp]
    L.fh_encode_bwd_ex.argtypes = [vp, vp, i64, vp, vp, ctypes.c_uint, vp]
    L.fh_encode_bwd_ex.restype = c_int
    L.fh_zero_grad.argtypes = [vp, vp, vp]
    L.fh_build_mhe.argtypes = [ctypes.POINTER(ctypes.c_uint32), c_int, c_int, c_int, u64, ctypes.c_uint32,
                               ctypes.POINTER(vp)]
    L.fh_build_mhe.restype = c_int
    L.fh_encoder_kind.argtypes = [vp]
    L.fh_level_stats_workspace_size.argtypes = [vp, c_int]
    L.fh_level_stats_workspace_size.restype = ctypes.c_size_t
    L.fh_level_stats.argtypes = [vp, c_int, vp, ctypes.c_size_t, vp, vp]
    L.fh_level_stats.restype = c_int
    L.fh_kernel_launches.argtypes = []
    L.fh_kernel_launches.restype = ctypes.c_ulonglong
    L.fh_encoder_scratch_size.argtypes = [vp]
    L.fh_encoder_scratch_size.restype = ctypes.c_size_t
    L.fh_encoder_attach_scratch.argtypes = [vp, vp, vp, ctypes.c_size_t]
    L.fh_encoder_attach_scratch.restype = c_int
    L.fh_encode_step_host.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp]
    L.fh_status_sync.argtypes = [vp, vp]
    L.fh_bench_gather.argtypes = [vp, u64, c_int, i64, c_int, c_int, ctypes.c_uint32, vp, vp]
    L.fh_bench_red.argtypes = [vp, u64, c_int, i64, c_int, c_int, ctypes.c_uint32, vp]
    L.fh_bench_copy.argtypes = [vp, vp, u64, vp]
    L.fh_bench_gather_levels.argtypes = [vp, vp, vp, c_int, c_int, i64, ctypes.c_uint32, vp, vp]
    L.fh_bench_red_levels.argtypes = [vp, vp, vp, c_int, c_int, i64, ctypes.c_uint32, vp]
    for name in ("fh_bench_gather", "fh_bench_red", "fh_bench_copy", "fh_bench_gather_levels", "fh_bench_red_levels"):
        getattr(L, name).restype = c_int
    L.fh_last_error.restype = ctypes.c_char_p
    L.fh_version.restype = ctypes.c_char_p
    for name in ("fh_fold_schedule", "fh_build_levels", "fh_level_info_get", "fh_encode_fwd", "fh_encode_bwd",
                 "fh_encode_indices", "fh_encode_fwd_bwd", "fh_encode_step_host", "fh_status_sync", "fh_zero_grad"):
        getattr(L, name).restype = c_int
    _lib = L
    return L


def _check(status: int):
    if status != FH_OK:
        raise FHashError(status, lib().fh_last_error().decode())


def _stream(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def fold_schedule(S_xyz: Sequence[int], n_t: int, fold: int) -> List[Tuple[int, int, int, int]]:
    """Eqs. 4-8 through the library; paper order (finest first)."""
    S = (ctypes.c_uint32 * 3)(*S_xyz)
    out = (LevelRes * 64)()
    L = ctypes.c_int(64)
    _check(lib().fh_fold_schedule(S, n_t, fold, out, ctypes.byref(L)))
    return [tuple(out[i].res) for i in range(L.value)]


_DT = {"f32": FH_F32, "f16": FH_F16, "bf16": FH_BF16}


FH_LIN_EQ9, FH_LIN_BRICK = 0, 1


class Encoder:
    """Handle on an fh_encoder (a1 build_levels).  levels: [(Rx,Ry,Rz,Rt)]
    in output order; cap 0 = pure MPHF; lin: FH_LIN_EQ9 (Eq. 9) or
    FH_LIN_BRICK (NEXT-2 brick order of the bijective levels, R21)."""

    def __init__(self, levels: Sequence[Sequence[int]], F: int, table_dtype: str = "f32", cap: int = 0,
                 lin: int = FH_LIN_EQ9, auto_scratch: bool = True):
        # auto_scratch: the binding allocates (torch) and attaches the
        # caller-owned shifted-pair scratch of each stream on that stream's
        # first pass (fh_encoder_attach_scratch); the library never allocates
        self._scratch = {}
        self.auto_scratch = auto_scratch
        L = len(levels)
        arr = (LevelRes * max(L, 1))()
        for i, r in enumerate(levels):
            arr[i].res[:] = [int(v) for v in r]
        h = ctypes.c_void_p()
        _check(lib().fh_build_levels_lin(arr, L, F, _DT[table_dtype], cap, lin, ctypes.byref(h)))
        self._h = h
        self.lin = lin
        self.levels = [tuple(int(v) for v in r) for r in levels]
        self.L, self.F, self.cap, self.table_dtype = L, F, cap, table_dtype
        self.entries = int(lib().fh_table_entries(h))
        self.param_count = int(lib().fh_param_count(h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.fh_encoder_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def level_info(self, l: int) -> dict:
        I = LevelInfo()
        _check(lib().fh_level_info_get(self._h, l, ctypes.byref(I)))
        return dict(res=tuple(I.res), corners=I.corners, table_size=I.table_size, hashed=bool(I.hashed),
                    offset=I.offset, lin=int(I.lin))

    def _auto_scratch(self, stream, device=None):
        """Attach torch-allocated scratch to `stream` once (see __init__)."""
        sid = _stream(stream)
        if not self.auto_scratch or sid in self._scratch:
            return
        import torch
        n = self.scratch_size()
        buf = None
        if n > 0:
            buf = torch.empty(n, dtype=torch.uint8, device=device or torch.device("cuda", torch.cuda.current_device()))
            _check(lib().fh_encoder_attach_scratch(self._h, sid, _ptr(buf), n))
        self._scratch[sid] = buf

    # -------------------------------------------------------------- kernels
    def fwd(self, coords, table, out=None, out_dtype: str = "f32", stream=None):
        import torch
        N = coords.shape[0]
        self._auto_scratch(stream, coords.device)
        if out is None:
            dt = torch.float32 if out_dtype == "f32" else torch.bfloat16
            out = torch.empty((N, self.L * self.F), dtype=dt, device=coords.device)
        _check(lib().fh_encode_fwd(self._h, _ptr(coords), N, _ptr(table), _ptr(out), _DT[out_dtype],
                                   _stream(stream)))
        return out

    def bwd(self, coords, dout, dtable, stream=None, overwrite: bool = False, level_major: bool = False):
        """dtable += gradient (fh_encode_bwd), or dtable = gradient with
        overwrite=True (fh_encode_bwd_ex FH_BWD_OVERWRITE: zeroed per level
        group right before its reductions).  level_major=True: dout is
        [L][N][F] (FH_BWD_DOUT_LEVEL_MAJOR) instead of [N][L*F]."""
        self._auto_scratch(stream, coords.device)
        if overwrite or level_major:
            flags = (1 if overwrite else 0) | (2 if level_major else 0)
            _check(lib().fh_encode_bwd_ex(self._h, _ptr(coords), coords.shape[0], _ptr(dout), _ptr(dtable), flags,
                                          _stream(stream)))
        else:
            _check(lib().fh_encode_bwd(self._h, _ptr(coords), coords.shape[0], _ptr(dout), _ptr(dtable),
                                       _stream(stream)))
        return dtable

    def indices(self, coords, want_w: bool = True, stream=None):
        import torch
        N = coords.shape[0]
        idx = torch.empty((N, self.L, 16), dtype=torch.int32, device=coords.device)
        w = torch.empty((N, self.L, 16), dtype=torch.float32, device=coords.device) if want_w else None
        _check(lib().fh_encode_indices(self._h, _ptr(coords), N, _ptr(idx), _ptr(w), _stream(stream)))
        return idx, w

    def level_stats(self, l: int, stream=None):
        """encoding_stats of level l on the GPU (fh_level_stats): (distinct
        buckets, collisions, utilisation) -- same tuple as the oracle's."""
        import torch
        L = lib()
        ws = int(L.fh_level_stats_workspace_size(self._h, l))
        w = torch.empty(ws, dtype=torch.uint8, device="cuda")
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
        _check(L.fh_level_stats(self._h, l, _ptr(w), ws, _ptr(out), _stream(stream)))
        d = int(out.item())
        info = self.level_info(l)
        if isinstance(self, MHEEncoder):
            C, T = info["res"][0] ** 3, self.T
        else:
            C, T = info["corners"], info["table_size"]
        return d, C - d, d / T

    def scratch_size(self) -> int:
        return int(lib().fh_encoder_scratch_size(self._h))

    def attach_scratch(self, buf, stream=None):
        """Use caller-owned device memory (>= scratch_size() bytes) as the
        shifted-pair scratch of `stream`; buf=None detaches (the stream then
        runs without the shifted pairs; no automatic re-attach)."""
        sid = _stream(stream)
        if buf is None:
            _check(lib().fh_encoder_attach_scratch(self._h, sid, None, 0))
        else:
            _check(lib().fh_encoder_attach_scratch(self._h, sid, _ptr(buf), buf.numel() * buf.element_size()))
        self._scratch[sid] = buf

    def zero_grad(self, dtable, stream=None):
        _check(lib().fh_zero_grad(self._h, _ptr(dtable), _stream(stream)))

    def fwd_bwd(self, coords, table, out, dout, dtable, out_dtype: str = "f32", zero_dtable: bool = True,
                stream=None):
        self._auto_scratch(stream, coords.device)
        _check(lib().fh_encode_fwd_bwd(self._h, _ptr(coords), coords.shape[0], _ptr(table), _ptr(out),
                                       _DT[out_dtype], _ptr(dout), _ptr(dtable), int(zero_dtable),
                                       _stream(stream)))

    def step_host(self, coords_h, dout_h, table_d, coords_d, dout_d, out_d, dtable_d, out_h, dtable_h,
                  stream=None):
        self._auto_scratch(stream, coords_d.device)
        _check(lib().fh_encode_step_host(self._h, _ptr(coords_h), _ptr(dout_h), coords_h.shape[0], _ptr(table_d),
                                         _ptr(coords_d), _ptr(dout_d), _ptr(out_d), _ptr(dtable_d), _ptr(out_h),
                                         _ptr(dtable_h), _stream(stream)))

    def status_sync(self, stream=None) -> int:
        """Synchronise and return the sticky status (FH_OK or FH_E_DOMAIN);
        raises on CUDA errors."""
        s = lib().fh_status_sync(self._h, _stream(stream))
        if s not in (FH_OK, FH_E_DOMAIN):
            _check(s)
        return s


# ------------------------------------------------------------ measurement
def bench_gather(buf, n_entries: int, entry_bytes: int, n_threads: int, sink, mode: int = 1, seed: int = 0,
                 stream=None):
    """Roofline microbenchmark (include/fhash_bench.h): 8 random x-pairs per
    thread; mode 1 = one aligned access per pair (minimum sectors)."""
    _check(lib().fh_bench_gather(_ptr(buf), n_entries, entry_bytes, n_threads, 8, mode, seed, _ptr(sink),
                                 _stream(stream)))


def bench_red(buf, n_entries: int, entry_bytes: int, n_threads: int, mode: int = 1, seed: int = 0, stream=None):
    _check(lib().fh_bench_red(_ptr(buf), n_entries, entry_bytes, n_threads, 8, mode, seed, _stream(stream)))


def _level_arrays(enc):
    off = (ctypes.c_uint64 * enc.L)(*[enc.level_info(l)["offset"] for l in range(enc.L)])
    size = (ctypes.c_uint64 * enc.L)(*[enc.level_info(l)["table_size"] for l in range(enc.L)])
    return off, size


def bench_gather_levels(buf, enc, entry_bytes: int, n_samples: int, sink, seed: int = 0, stream=None):
    """Level-mix roofline microbenchmark: the encode's thread shape (sample,
    level), 8 ideal x-pairs per thread inside each level's table range."""
    off, size = _level_arrays(enc)
    _check(lib().fh_bench_gather_levels(_ptr(buf), off, size, enc.L, entry_bytes, n_samples, seed, _ptr(sink),
                                        _stream(stream)))


def bench_red_levels(buf, enc, entry_bytes: int, n_samples: int, seed: int = 0, stream=None):
    off, size = _level_arrays(enc)
    _check(lib().fh_bench_red_levels(_ptr(buf), off, size, enc.L, entry_bytes, n_samples, seed, _stream(stream)))


def kernel_launches() -> int:
    """Kernels the library has launched so far (fh_kernel_launches)."""
    return int(lib().fh_kernel_launches())


def bench_copy(dst, src, nbytes: int, stream=None):
    _check(lib().fh_bench_copy(_ptr(dst), _ptr(src), nbytes, _stream(stream)))


# ------------------------------------------------------------ train step
class MLPDesc(ctypes.Structure):
    _fields_ = [("n_in", ctypes.c_int), ("n_hidden", ctypes.c_int), ("n_hidden_layers", ctypes.c_int)]


class TrainBuffers(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("table_master", "table_shadow", "table_grad", "table_m", "table_v",
                                               "mlp_master", "mlp_shadow", "mlp_grad", "mlp_m", "mlp_v",
                                               "workspace")] + [("workspace_bytes", ctypes.c_size_t)]


class AdamCfg(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double)]


def _train_lib():
    L = lib()
    if getattr(L, "_train_ready", False):
        return L
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    L.fh_mlp_param_count.argtypes = [ctypes.POINTER(MLPDesc)]
    L.fh_mlp_param_count.restype = ctypes.c_uint64
    L.fh_train_workspace_size.argtypes = [vp, ctypes.POINTER(MLPDesc), i64]
    L.fh_train_workspace_size.restype = ctypes.c_size_t
    L.fh_trainer_create.argtypes = [vp, ctypes.POINTER(MLPDesc), ctypes.POINTER(TrainBuffers),
                                    ctypes.POINTER(AdamCfg), i64, ctypes.POINTER(vp)]
    L.fh_train_fwd_bwd.argtypes = [vp, vp, vp, i64, i64, vp, vp]
    L.fh_train_step.argtypes = [vp, vp, vp, i64, i64, vp, vp]
    L.fh_train_apply.argtypes = [vp, vp]
    L.fh_train_apply_sharded.argtypes = [vp, i64, i64, vp, vp]
    L.fh_train_apply_sharded.restype = ctypes.c_int
    L.fh_train_dx_layout.argtypes = [vp]
    L.fh_train_dx_layout.restype = ctypes.c_int
    L.fh_train_bwd_launches.argtypes = [vp]
    L.fh_train_bwd_launches.restype = ctypes.c_int
    L.fh_train_bwd_ranges.argtypes = [vp, ctypes.c_int, ctypes.POINTER(i64), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    L.fh_train_bwd_ranges.restype = ctypes.c_int
    L.fh_train_set_bwd_events.argtypes = [vp, ctypes.POINTER(vp), ctypes.c_int]
    L.fh_train_set_bwd_events.restype = ctypes.c_int
    L.fh_train_apply_ranges.argtypes = [vp, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                        ctypes.POINTER(vp), vp]
    L.fh_train_apply_ranges.restype = ctypes.c_int
    L.fh_train_apply_peers.argtypes = [vp, ctypes.c_int, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                       ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                       ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int, vp]
    L.fh_train_apply_peers.restype = ctypes.c_int
    L.fh_train_apply_multicast.argtypes = [vp, vp, vp, vp, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                           ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int, vp]
    L.fh_train_apply_multicast.restype = ctypes.c_int
    L.fh_nccl_unique_id.argtypes = [vp]
    L.fh_nccl_comm_create.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    L.fh_nccl_comm_destroy.argtypes = [vp]
    L.fh_trainer_dp_workspace_size.argtypes = [vp, ctypes.c_int]
    L.fh_trainer_dp_workspace_size.restype = ctypes.c_size_t
    L.fh_trainer_set_comm.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_size_t]
    for n in ("fh_nccl_unique_id", "fh_nccl_comm_create", "fh_nccl_comm_destroy", "fh_trainer_set_comm"):
        getattr(L, n).restype = ctypes.c_int
    L.fh_infer_workspace_size.argtypes = [vp, ctypes.POINTER(MLPDesc), i64]
    L.fh_infer_workspace_size.restype = ctypes.c_size_t
    L.fh_infer.argtypes = [vp, ctypes.POINTER(MLPDesc), vp, vp, vp, vp, i64, vp, vp, ctypes.c_size_t, vp]
    L.fh_infer.restype = ctypes.c_int
    L.fh_arm_pace.argtypes = [i64, i64]
    L.fh_arm_pace.restype = i64
    L.fh_trainer_status.argtypes = [vp, vp]
    L.fh_trainer_step_count.argtypes = [vp]
    L.fh_trainer_step_count.restype = i64
    L.fh_trainer_destroy.argtypes = [vp]
    L.fh_trainer_destroy.restype = None
    for n in ("fh_trainer_create", "fh_train_fwd_bwd", "fh_train_step", "fh_train_apply", "fh_trainer_status"):
        getattr(L, n).restype = ctypes.c_int
    L._train_ready = True
    return L


class Trainer:
    """Handle on an fh_trainer plus the device buffers it trains (torch
    tensors on the current device; allocation only).

    grads: ONE flat fp32 tensor [table (padded to 4) | mlp] so that a data
    parallel caller all-reduces a single buffer between fwd_bwd() and
    apply()."""

    def __init__(self, enc: "Encoder", table_init, mlp_layers, max_batch: int, lr: float = 0.01,
                 beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, world: int = 1, alloc=None):
        # world > 1: the flat table region of grads and shadow is padded to a
        # multiple of 4 * world so it splits into equal 16-byte-aligned shards
        # (reduce-scatter / sharded Adam / all-gather, dp.sharded_step).
        # alloc(numel, dtype, device): allocator of the grads and shadow
        # buffers (e.g. torch symmetric memory for dp.PeerShardedDP).
        import numpy as np
        import torch
        L = _train_lib()
        self.enc = enc
        self.K0 = enc.L * enc.F
        self.desc = MLPDesc(self.K0, 64, 2)
        dev = torch.device("cuda", torch.cuda.current_device())
        nt = enc.entries * enc.F
        q = 4 * max(1, world)
        nt_pad = (nt + q - 1) // q * q
        self.world, self.nt_pad = max(1, world), nt_pad
        P = int(L.fh_mlp_param_count(ctypes.byref(self.desc)))
        self.n_table, self.n_mlp = nt, P
        f32 = dict(dtype=torch.float32, device=dev)
        if isinstance(table_init, torch.Tensor):
            self.table_master = table_init.to(device=dev, dtype=torch.float32).reshape(enc.entries, enc.F).contiguous()
        else:
            self.table_master = torch.as_tensor(np.asarray(table_init, dtype=np.float32)).reshape(
                enc.entries, enc.F).to(dev)
        self.table_shadow, self.shadow_flat = None, None
        def zeros(n, dtype):
            if alloc is None:
                return torch.zeros(n, dtype=dtype, device=dev)
            t = alloc(n, dtype, dev)
            t.zero_()
            return t
        if enc.table_dtype == "f16":
            self.shadow_flat = zeros(nt_pad, torch.float16)
            self.shadow_flat[:nt].copy_(self.table_master.view(-1))
            self.table_shadow = self.shadow_flat[:nt].view(enc.entries, enc.F)
        self.grads = zeros(nt_pad + P, torch.float32)
        self.table_grad = self.grads[:nt].view(enc.entries, enc.F)
        self.mlp_grad = self.grads[nt_pad:]
        self.table_m = torch.zeros(nt, **f32)
        self.table_v = torch.zeros(nt, **f32)
        flat = []
        for W, b in mlp_layers:
            flat += [np.asarray(W, np.float32).ravel(), np.asarray(b, np.float32).ravel()]
        flat = np.concatenate(flat)
        assert flat.size == P, (flat.size, P)
        self.mlp_master = torch.from_numpy(flat).to(dev)
        self.mlp_shadow = self.mlp_master.bfloat16()
        self.mlp_m = torch.zeros(P, **f32)
        self.mlp_v = torch.zeros(P, **f32)
        ws = int(L.fh_train_workspace_size(enc.handle, ctypes.byref(self.desc), max_batch))
        self.workspace = torch.zeros(ws, dtype=torch.uint8, device=dev)
        self.max_batch = max_batch
        b = TrainBuffers(self.table_master.data_ptr(), _ptr(self.table_shadow), self.table_grad.data_ptr(),
                         self.table_m.data_ptr(), self.table_v.data_ptr(), self.mlp_master.data_ptr(),
                         self.mlp_shadow.data_ptr(), self.mlp_grad.data_ptr(), self.mlp_m.data_ptr(),
                         self.mlp_v.data_ptr(), self.workspace.data_ptr(), ws)
        self._bufs = b
        adam = AdamCfg(lr, beta1, beta2, eps)
        h = ctypes.c_void_p()
        _check(L.fh_trainer_create(enc.handle, ctypes.byref(self.desc), ctypes.byref(b), ctypes.byref(adam),
                                   max_batch, ctypes.byref(h)))
        self._h = h
        self.loss = torch.zeros(1, **f32)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.fh_trainer_destroy(h)
            self._h = None

    # workspace views (read-only use in tests)
    def enc_out(self, N):
        import torch
        return self.workspace[: N * self.K0 * 2].view(torch.bfloat16).view(N, self.K0)

    def dx_layout(self):
        """0: dL/d(enc) row-major [N][K0]; F: level-major [L][N][F] (fh_train_dx_layout)."""
        return int(_train_lib().fh_train_dx_layout(self._h))

    def dx_raw(self, N):
        """The dL/d(enc) workspace of an N-sample step as stored (flat f32)."""
        import torch
        off = ((self.max_batch + 7) // 8 * 8 * self.K0 * 2 + 255) // 256 * 256   # encoder rows in whole 8-row groups
        return self.workspace[off: off + N * self.K0 * 4].view(torch.float32)

    def dx(self, N):
        """dL/d(enc) as [N][K0] (a permuted copy when stored level-major)."""
        F = self.dx_layout()
        raw = self.dx_raw(N)
        if F > 0:
            return raw.view(self.K0 // F, N, F).permute(1, 0, 2).reshape(N, self.K0)
        return raw.view(N, self.K0)

    def fwd_bwd(self, coords, target, n_global=None, stream=None):
        N = coords.shape[0]
        self.enc._auto_scratch(stream, coords.device)
        _check(_train_lib().fh_train_fwd_bwd(self._h, _ptr(coords), _ptr(target), N, n_global or N,
                                             self.loss.data_ptr(), _stream(stream)))
        return self.loss

    def infer(self, coords, y=None, stream=None):
        """Model evaluation V = model(S) (fh_infer) with this trainer's
        current parameters; reuses the trainer workspace's encoder buffer."""
        import torch
        N = coords.shape[0]
        assert N <= self.max_batch
        if y is None:
            y = torch.empty(N, dtype=torch.float32, device=coords.device)
        table = self.table_shadow if self.table_shadow is not None else self.table_master
        self.enc._auto_scratch(stream, coords.device)
        L = _train_lib()
        ws = int(L.fh_infer_workspace_size(self.enc.handle, ctypes.byref(self.desc), N))
        _check(L.fh_infer(self.enc.handle, ctypes.byref(self.desc), _ptr(table), _ptr(self.mlp_shadow),
                          _ptr(self.mlp_master), _ptr(coords), N, _ptr(y), _ptr(self.workspace), ws,
                          _stream(stream)))
        return y

    def apply_sharded(self, begin: int, end: int, grad_shard, stream=None):
        _check(_train_lib().fh_train_apply_sharded(self._h, begin, end, _ptr(grad_shard), _stream(stream)))

    def apply(self, stream=None):
        _check(_train_lib().fh_train_apply(self._h, _stream(stream)))

    # -- overlap of the gradient reduction with the backward (dp.OverlappedShardedDP)
    def bwd_launch_ranges(self):
        """[[(begin, end), ...] per backward launch] in flat table elements."""
        L = _train_lib()
        n = int(L.fh_train_bwd_launches(self._h))
        if n < 0:
            raise FHashError(FH_E_STATE, "fh_train_bwd_launches failed")
        out = []
        for i in range(n):
            buf = (ctypes.c_int64 * 64)()
            k = ctypes.c_int()
            _check(L.fh_train_bwd_ranges(self._h, i, buf, 32, ctypes.byref(k)))
            out.append([(int(buf[2 * j]), int(buf[2 * j + 1])) for j in range(k.value)])
        return out

    def set_bwd_events(self, events):
        """events: torch.cuda.Event list (one per backward launch) or []."""
        arr = (ctypes.c_void_p * max(1, len(events)))(*[e.cuda_event for e in events])
        self._events = list(events)   # keep alive
        _check(_train_lib().fh_train_set_bwd_events(self._h, arr, len(events)))

    def apply_peers(self, peer_grads, peer_shadows, peer_mlp_grads, ranges, broadcast, with_mlp, new_step,
                    stream=None):
        """fh_train_apply_peers: peer_* are lists of W device addresses (int)."""
        W, n = len(peer_grads), len(ranges)
        pg = (ctypes.c_void_p * W)(*peer_grads)
        ps = (ctypes.c_void_p * W)(*peer_shadows)
        pm = (ctypes.c_void_p * W)(*peer_mlp_grads)
        b = (ctypes.c_int64 * max(1, n))(*[r[0] for r in ranges])
        e = (ctypes.c_int64 * max(1, n))(*[r[1] for r in ranges])
        bc = (ctypes.c_int * max(1, n))(*[int(x) for x in broadcast])
        _check(_train_lib().fh_train_apply_peers(self._h, W, pg, ps, pm, n, b, e, bc, int(with_mlp), int(new_step),
                                                 _stream(stream)))

    def apply_multicast(self, mc_grads, mc_shadow, mc_mlp_grads, ranges, broadcast, with_mlp, new_step,
                        stream=None):
        """fh_train_apply_multicast: mc_* are NVLS multicast device addresses (int)."""
        n = len(ranges)
        b = (ctypes.c_int64 * max(1, n))(*[r[0] for r in ranges])
        e = (ctypes.c_int64 * max(1, n))(*[r[1] for r in ranges])
        bc = (ctypes.c_int * max(1, n))(*[int(x) for x in broadcast])
        _check(_train_lib().fh_train_apply_multicast(self._h, mc_grads, mc_shadow, mc_mlp_grads, n, b, e, bc,
                                                     int(with_mlp), int(new_step), _stream(stream)))

    def apply_ranges(self, ranges, grads, stream=None):
        """One Adam step over table element ranges [(b, e)] with grads (f32
        CUDA tensors of e-b values each) + the MLP segment."""
        n = len(ranges)
        b = (ctypes.c_int64 * max(1, n))(*[r[0] for r in ranges])
        e = (ctypes.c_int64 * max(1, n))(*[r[1] for r in ranges])
        g = (ctypes.c_void_p * max(1, n))(*[t.data_ptr() for t in grads])
        _check(_train_lib().fh_train_apply_ranges(self._h, n, b, e, g, _stream(stream)))

    def step(self, coords, target, n_global=None, stream=None):
        N = coords.shape[0]
        self.enc._auto_scratch(stream, coords.device)
        _check(_train_lib().fh_train_step(self._h, _ptr(coords), _ptr(target), N, n_global or N,
                                          self.loss.data_ptr(), _stream(stream)))
        return self.loss

    def set_comm(self, comm: "NcclComm"):
        """The fused data-parallel form (fh_trainer_set_comm): from now on
        step() reduce-scatters / all-reduces / all-gathers through `comm`
        inside the library.  comm=None detaches."""
        import torch
        L = _train_lib()
        if comm is None:
            _check(L.fh_trainer_set_comm(self._h, None, 1, 0, None, 0))
            self._dp_ws = None
            return
        n = int(L.fh_trainer_dp_workspace_size(self._h, comm.nranks))
        self._dp_ws = torch.empty(max(n, 256), dtype=torch.uint8, device=self.grads.device)
        self._comm = comm   # keep alive
        _check(L.fh_trainer_set_comm(self._h, comm.handle, comm.nranks, comm.rank, _ptr(self._dp_ws),
                                     self._dp_ws.numel()))

    def status(self, stream=None) -> int:
        s = _train_lib().fh_trainer_status(self._h, _stream(stream))
        if s not in (FH_OK, FH_E_DOMAIN, FH_E_DIVERGED):
            _check(s)
        return s

    @property
    def step_count(self) -> int:
        return int(_train_lib().fh_trainer_step_count(self._h))


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (fh_nccl_unique_id) for NcclComm; rank 0 makes
    it, the caller broadcasts it (e.g. torch.distributed.broadcast_object_list)."""
    buf = ctypes.create_string_buffer(128)
    _check(_train_lib().fh_nccl_unique_id(buf))
    return buf.raw


class NcclComm:
    """An NCCL communicator made by the library (fh_nccl_comm_create) from
    torch's libnccl, for Trainer.set_comm (the fused data-parallel form)."""

    def __init__(self, uid: bytes, nranks: int, rank: int):
        h = ctypes.c_void_p()
        _check(_train_lib().fh_nccl_comm_create(ctypes.create_string_buffer(uid, 128), nranks, rank, ctypes.byref(h)))
        self.handle, self.nranks, self.rank = h, nranks, rank

    def destroy(self):
        if self.handle is not None and self.handle.value:
            _check(_train_lib().fh_nccl_comm_destroy(self.handle))
        self.handle = None


def arm_pace(n_rays: int, n_alive: int) -> int:
    """Alg. 1 marching pace N_s = max(min(N_r / N_a, 64), 1) (fh_arm_pace)."""
    return int(_train_lib().fh_arm_pace(n_rays, n_alive))


# ------------------------------------------------------------ synthetic data (harness)
def _data_lib():
    L = lib()
    if getattr(L, "_data_ready", False):
        return L
    vp, c_int, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    L.fh_data_gaussian_blobs.argtypes = [vp, c_int, c_int, c_int, vp, vp]
    L.fh_data_value_noise.argtypes = [vp, c_int, c_int, c_int, c_int, ctypes.c_uint32, vp]
    L.fh_data_normalize.argtypes = [vp, i64, ctypes.c_float, vp, vp]
    L.fh_data_sample_voxels.argtypes = [vp, c_int, c_int, c_int, c_int, i64, ctypes.c_uint64, ctypes.c_uint32,
                                        ctypes.c_uint32, vp, vp, vp]
    for n in ("fh_data_gaussian_blobs", "fh_data_value_noise", "fh_data_normalize", "fh_data_sample_voxels"):
        getattr(L, n).restype = c_int
    L._data_ready = True
    return L


def field_gaussian_blobs(S: int, T: int, blobs, stream=None):
    """BASELINE.json configs[2] field on the device, normalised to [0,1].
    blobs: [n][7] float32 host array (sigma, c0xyz, vxyz)."""
    import numpy as np
    import torch
    b = np.ascontiguousarray(blobs, dtype=np.float32)
    f = torch.empty((T, S, S, S), dtype=torch.float32, device="cuda")
    scratch = torch.empty(16, dtype=torch.float32, device="cuda")
    L = _data_lib()
    _check(L.fh_data_gaussian_blobs(f.data_ptr(), S, T, b.shape[0], b.ctypes.data, _stream(stream)))
    _check(L.fh_data_normalize(f.data_ptr(), f.numel(), 0.0, scratch.data_ptr(), _stream(stream)))
    return f


def field_value_noise(Sx: int, Sy: int, Sz: int, T: int, seed: int = 0, band: float = 0.02, stream=None):
    """BASELINE.json configs[3] field on the device: 3-octave 4D value noise
    with a sharp isosurface band, normalised to [0,1]."""
    import torch
    f = torch.empty((T, Sz, Sy, Sx), dtype=torch.float32, device="cuda")
    scratch = torch.empty(16, dtype=torch.float32, device="cuda")
    L = _data_lib()
    _check(L.fh_data_value_noise(f.data_ptr(), Sx, Sy, Sz, T, seed, _stream(stream)))
    _check(L.fh_data_normalize(f.data_ptr(), f.numel(), band, scratch.data_ptr(), _stream(stream)))
    return f


def sample_voxels(field, N: int, seed: int, subsequence: int, offset: int, coords=None, target=None, stream=None):
    """Philox voxel sampler: returns (coords [N][4], target [N])."""
    import torch
    T, Sz, Sy, Sx = field.shape
    if coords is None:
        coords = torch.empty((N, 4), dtype=torch.float32, device=field.device)
    if target is None:
        target = torch.empty((N,), dtype=torch.float32, device=field.device)
    _check(_data_lib().fh_data_sample_voxels(field.data_ptr(), Sx, Sy, Sz, T, N, seed, subsequence, offset,
                                             coords.data_ptr(), target.data_ptr(), _stream(stream)))
    return coords, target


class MHEEncoder(Encoder):
    """NEXT-3: the MHE baseline encoder (fh_build_mhe) behind the same
    fwd / bwd / indices calls.  res: vertices per spatial axis per level."""

    def __init__(self, res: Sequence[int], F: int, T: int, n_frames: int, table_dtype: str = "f32"):
        self._scratch = {}
        self.auto_scratch = False   # MHE encoders use no scratch
        L = len(res)
        arr = (ctypes.c_uint32 * max(L, 1))(*[int(r) for r in res])
        h = ctypes.c_void_p()
        _check(lib().fh_build_mhe(arr, L, F, _DT[table_dtype], T, n_frames, ctypes.byref(h)))
        self._h = h
        self.levels = [(int(r), int(r), int(r), int(n_frames)) for r in res]
        self.L, self.F, self.cap, self.table_dtype = L, F, T, table_dtype
        self.T, self.n_frames = T, n_frames
        self.entries = int(lib().fh_table_entries(h))
        self.param_count = int(lib().fh_param_count(h))

    def indices(self, coords, want_w: bool = True, stream=None):
        import torch
        N = coords.shape[0]
        idx = torch.empty((N, self.L, 8), dtype=torch.int32, device=coords.device)
        w = torch.empty((N, self.L, 8), dtype=torch.float32, device=coords.device) if want_w else None
        _check(lib().fh_encode_indices(self._h, _ptr(coords), N, _ptr(idx), _ptr(w), _stream(stream)))
        return idx, w


# ------------------------------------------------------------ NEXT-4 coreset
FH_FEAT_INTERVAL, FH_FEAT_ISOSURFACE, FH_FEAT_SEGMENTATION = 0, 1, 2


class FeatureSpec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("p0", ctypes.c_float), ("p1", ctypes.c_float)]


def _coreset_lib():
    L = lib()
    if getattr(L, "_coreset_ready", False):
        return L
    vp, u32p, i64 = ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32), ctypes.c_int64
    L.fh_coreset_workspace_size.argtypes = [u32p, ctypes.c_int]
    L.fh_coreset_workspace_size.restype = ctypes.c_size_t
    L.fh_occupancy_words.argtypes = [u32p]
    L.fh_occupancy_words.restype = ctypes.c_uint64
    L.fh_morton_cell.argtypes = [u32p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
    L.fh_morton_cell.restype = ctypes.c_uint64
    L.fh_coreset_build.argtypes = [vp, u32p, ctypes.c_int, ctypes.POINTER(FeatureSpec), vp, ctypes.c_size_t, vp,
                                   vp, vp, vp]
    L.fh_coreset_build.restype = ctypes.c_int
    L.fh_coreset_emit.argtypes = [vp, u32p, ctypes.c_int, vp, ctypes.c_size_t, vp, vp, ctypes.c_uint64, vp]
    L.fh_coreset_emit.restype = ctypes.c_int
    L._coreset_ready = True
    return L


def occupancy_words(dims_xyz) -> int:
    return int(_coreset_lib().fh_occupancy_words((ctypes.c_uint32 * 3)(*dims_xyz)))


def morton_cell(dims_xyz, x: int, y: int, z: int) -> int:
    return int(_coreset_lib().fh_morton_cell((ctypes.c_uint32 * 3)(*dims_xyz), x, y, z))


class Coreset:
    """NEXT-4: feature-based coreset selection (fh_coreset_build / _emit) on
    the key frames vol [n][Z][Y][X] float32 (a CUDA tensor).  build() is
    stream-ordered; .count / .fbb synchronise to read the results."""

    def __init__(self, vol, kind: int, p0: float, p1: float = 0.0, occupancy: bool = True, stream=None):
        import torch
        n, Z, Y, X = vol.shape
        self.vol, self.n = vol, n
        self.dims = (ctypes.c_uint32 * 3)(X, Y, Z)
        L = _coreset_lib()
        ws = int(L.fh_coreset_workspace_size(self.dims, n))
        if ws == 0:
            raise FHashError(FH_E_RANGE, "coreset: volume too large or degenerate")
        dev = vol.device
        self.workspace = torch.empty(ws, dtype=torch.uint8, device=dev)
        self.fbb_dev = torch.empty(6, dtype=torch.int32, device=dev)
        self.count_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        self.words = int(L.fh_occupancy_words(self.dims))
        self.occupancy = torch.empty((n, self.words), dtype=torch.int32, device=dev) if occupancy else None
        self.spec = FeatureSpec(kind, p0, p1)
        _check(L.fh_coreset_build(_ptr(vol), self.dims, n, ctypes.byref(self.spec), _ptr(self.workspace), ws,
                                  _ptr(self.occupancy), _ptr(self.fbb_dev), _ptr(self.count_dev), _stream(stream)))

    @property
    def count(self) -> int:
        return int(self.count_dev.item())

    @property
    def fbb(self):
        f = self.fbb_dev.cpu().tolist()
        return None if f[0] == 2 ** 31 - 1 else (tuple(f[:3]), tuple(f[3:]))

    def emit(self, coords=None, values=None, stream=None):
        import torch
        M = self.count
        if coords is None:
            coords = torch.empty((max(M, 1), 4), dtype=torch.float32, device=self.vol.device)
        if values is None:
            values = torch.empty((max(M, 1),), dtype=torch.float32, device=self.vol.device)
        cap = min(coords.shape[0], values.shape[0])
        _check(_coreset_lib().fh_coreset_emit(_ptr(self.vol), self.dims, self.n, _ptr(self.workspace),
                                              self.workspace.numel(), _ptr(coords), _ptr(values), cap,
                                              _stream(stream)))
        return coords[:M], values[:M]
