"""paper_2403_10266_b200 — B200-native Dynamic Sequence Parallelism hot path.

Thin ctypes binding over libdsp.so (include/dsp.h, include/dsp_kernels.h): every
function here only marshals arguments (torch tensors -> device pointers, the current
CUDA stream) and calls the C ABI of the same name; every step of the path runs in the
library's CUDA kernels or NCCL.  There is no CPU fallback: if the library is missing
or a tensor is not on a CUDA device, calls raise.

Paper: arXiv 2403.10266 (DSP).  The block forward is §3.1: spatial
attention local on T-shards -> dynamic switch (one all-to-all) -> temporal attention
+ MLP local on S-shards -> switch back ("two AlltoAll operations in total").
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DSP_LIB_OVERRIDE") or os.path.join(_HERE, "libdsp.so")  # override: A/B experiments only

DSP_DIM_T, DSP_DIM_S = 1, 2
DSP_BF16, DSP_F32 = 0, 1
DSP_SWITCH_NCCL, DSP_SWITCH_P2P, DSP_SWITCH_FUSED = 0, 1, 2
DSP_EPI_NONE, DSP_EPI_RESIDUAL, DSP_EPI_GELU = 0, 1, 2
IMPLS = {"nccl": DSP_SWITCH_NCCL, "p2p": DSP_SWITCH_P2P, "fused": DSP_SWITCH_FUSED}
DIMS = {"T": DSP_DIM_T, "S": DSP_DIM_S, DSP_DIM_T: DSP_DIM_T, DSP_DIM_S: DSP_DIM_S}

STATUS = {0: "DSP_OK", 1: "DSP_ERR_NULL", 2: "DSP_ERR_SHAPE", 3: "DSP_ERR_DIVISIBILITY", 4: "DSP_ERR_SAME_DIM",
          5: "DSP_ERR_BAD_DIM", 6: "DSP_ERR_UNSUPPORTED", 7: "DSP_ERR_ALIGNMENT", 8: "DSP_ERR_ALIAS",
          9: "DSP_ERR_WORKSPACE", 10: "DSP_ERR_CUDA", 11: "DSP_ERR_NCCL", 12: "DSP_ERR_STATE",
          13: "DSP_ERR_PEER_TIMEOUT"}
SIGNAL_PAD_BYTES = 128  # DSP_SIGNAL_PAD_BYTES (include/dsp.h)


class DSPError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class Shape(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int64), ("T", ctypes.c_int64), ("S", ctypes.c_int64), ("C", ctypes.c_int64),
                ("num_heads", ctypes.c_int32), ("dtype", ctypes.c_int)]


CROSS_NAMES = ("ln_c_w", "ln_c_b", "w_q_c", "w_kv_c", "w_o_c")
LATTE_NAMES = ("ln_m_w", "ln_m_b", "w_fc1_s", "w_fc2_s")  # the Latte pair's spatial MLP (R38)
ADALN_SUBLAYERS = ("s", "t", "m", "ms")  # dsp_adaln_fold's mod rows: spatial attn, temporal attn, MLP, spatial MLP


class BlockWeights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("ln1_w", "ln1_b", "w_qkv_s", "w_o_s", "ln2_w", "ln2_b", "w_qkv_t",
                                               "w_o_t", "ln3_w", "ln3_b", "w_fc1", "w_fc2")] + [
        ("ln_eps", ctypes.c_float), ("prepared", ctypes.c_void_p)] + [
        (n, ctypes.c_void_p) for n in CROSS_NAMES] + [("ctx_tokens", ctypes.c_void_p), ("ctx_len", ctypes.c_int64)] + [
        (n, ctypes.c_void_p) for n in LATTE_NAMES] + [("pe_t", ctypes.c_void_p)]


GRAD_NAMES = ("ln1_w", "ln1_b", "w_qkv_s", "w_o_s", "ln2_w", "ln2_b", "w_qkv_t", "w_o_t", "ln3_w", "ln3_b",
              "w_fc1", "w_fc2")


class BlockGrads(ctypes.Structure):  # dsp_block_grads_t (include/dsp_train.h): fp32 accumulators
    _fields_ = [(n, ctypes.c_void_p) for n in GRAD_NAMES]


SAVED_NAMES = ("h1", "qkv_s", "o_s", "lse_s", "y1s", "h2", "qkv_t", "o_t", "lse_t", "y2", "h3", "u", "g")


class SavedLayout(ctypes.Structure):  # dsp_train_saved_layout_t
    _fields_ = [(n, ctypes.c_int64) for n in SAVED_NAMES + ("total",)]


class SwitchPlan(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64 * 3), ("run_bytes", ctypes.c_int64), ("src_stride", ctypes.c_int64 * 3),
                ("dst_stride", ctypes.c_int64 * 3), ("dst_peer_off", ctypes.c_int64),
                ("pack_is_identity", ctypes.c_int32), ("unpack_is_identity", ctypes.c_int32)]


class SwitchNdPlan(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64 * 4), ("run_bytes", ctypes.c_int64), ("src_stride", ctypes.c_int64 * 4),
                ("dst_stride", ctypes.c_int64 * 4), ("dst_peer_off", ctypes.c_int64),
                ("pack_is_identity", ctypes.c_int32), ("unpack_is_identity", ctypes.c_int32)]


class AttnWeights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("ln_w", "ln_b", "w_qkv", "w_o")]


class MlpWeights(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("ln_w", "ln_b", "w_fc1", "w_fc2")]


STAGES = ("LN1", "QKV_S", "ATTN_S", "PROJ_S", "SWITCH_TS", "LN2", "QKV_T", "ATTN_T", "PROJ_T", "LN3", "FC1",
          "FC2", "SWITCH_ST")
WEIGHT_NAMES = tuple(n for n, _ in BlockWeights._fields_[:12])

_lib = None


def lib() -> ctypes.CDLL:
    """Load libdsp.so (built in-tree by __graft_entry__.build()); raise if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2403_10266_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        P = ctypes.POINTER
        sig = {
            "dsp_ctx_create": [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, P(vp)],
            "dsp_ctx_destroy": [vp],
            "dsp_ctx_set_workspace": [vp, vp, ctypes.c_size_t],
            "dsp_ctx_set_peer_buffers": [vp, P(vp), P(vp), ctypes.c_size_t],
            "dsp_split": [vp, P(Shape), ctypes.c_int, vp, vp, vp],
            "dsp_gather": [vp, P(Shape), ctypes.c_int, vp, vp, vp],
            "dsp_switch": [vp, P(Shape), ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int, vp],
            "dsp_switch_volume": [P(Shape), ctypes.c_int, P(i64), P(i64)],
            "dsp_switch_plan": [P(Shape), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P(SwitchPlan)],
            "dsp_switch_nd_plan": [P(i64), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, P(SwitchNdPlan)],
            "dsp_switch_nd": [vp, P(i64), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int,
                              vp],
            "dsp_nd_block_forward": [vp, P(i64), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     P(ctypes.c_int), P(AttnWeights), P(MlpWeights), ctypes.c_float, ctypes.c_int, vp,
                                     vp, ctypes.c_int, vp],
            "dsp_cross_attn": [vp, P(Shape), vp, vp, i64, vp, vp, vp, vp, vp, vp],
            "dsp_spatial_attn": [vp, P(Shape), vp, vp, vp, vp, vp, vp],
            "dsp_temporal_attn": [vp, P(Shape), vp, vp, vp, vp, vp, vp],
            "dsp_st_block_forward": [vp, P(Shape), P(BlockWeights), vp, vp, ctypes.c_int, vp],
            "dsp_st_model_forward": [vp, P(Shape), P(P(BlockWeights)), ctypes.c_int, vp, vp, ctypes.c_int, vp],
            "dsp_st_block_forward_host": [vp, P(Shape), P(BlockWeights), vp, vp, vp, vp, ctypes.c_int, vp],
            "dsp_st_block_prepare": [vp, P(Shape), P(BlockWeights), vp, ctypes.c_size_t, vp],
            "dsp_adaln_fold": [vp, P(Shape), P(BlockWeights), vp, P(BlockWeights), vp],
            "dsp_st_block_forward_host_pipelined": [vp, P(Shape), P(BlockWeights), ctypes.c_int, P(vp), P(vp),
                                                    P(vp), P(vp), ctypes.c_int, vp],
            "dsp_layer_norm": [vp, ctypes.c_int, i64, i64, vp, vp, vp, ctypes.c_float, vp, vp],
            "dsp_linear": [vp, ctypes.c_int, i64, i64, i64, vp, vp, vp, ctypes.c_int, vp, vp],
            "dsp_attention_core": [vp, ctypes.c_int, i64, i64, i64, i64, i32, ctypes.c_int, vp, vp, vp],
            "dsp_ctx_set_stage_events": [vp, P(vp), ctypes.c_int],
            "dsp_switch_pack": [vp, P(Shape), ctypes.c_int, ctypes.c_int, vp, vp, vp],
            "dsp_switch_unpack": [vp, P(Shape), ctypes.c_int, ctypes.c_int, vp, vp, vp],
            "dsp_gather_unpack": [vp, P(Shape), ctypes.c_int, vp, vp, vp],
            "dsp_ctx_set_barrier_timeout": [vp, ctypes.c_double],
            "dsp_ctx_check_errors": [vp],
            "dsp_ctx_set_tap": [vp, ctypes.c_int, vp, ctypes.c_size_t],
            "dsp_ctx_set_stage_clocks": [vp, vp],
            "dsp_ctx_set_collective_emulation": [vp, ctypes.c_int],
            "dsp_st_block_forward_ulysses": [vp, P(Shape), P(BlockWeights), vp, vp, ctypes.c_int, vp],
            # training path (include/dsp_train.h)
            "dsp_train_saved_layout": [P(Shape), ctypes.c_int, P(SavedLayout)],
            "dsp_st_block_forward_train": [vp, P(Shape), P(BlockWeights), vp, vp, vp, ctypes.c_int, vp],
            "dsp_st_block_backward": [vp, P(Shape), P(BlockWeights), vp, vp, vp, vp, P(BlockGrads), ctypes.c_int,
                                      vp],
            "dsp_grads_reduce": [vp, vp, i64, ctypes.c_int, vp, vp],
            "dsp_linear_dgrad": [vp, i64, i64, i64, vp, vp, vp, vp, vp],
            "dsp_linear_wgrad": [vp, i64, i64, i64, vp, vp, vp, ctypes.c_int, vp],
            "dsp_linear_gelu_aux": [vp, i64, i64, i64, vp, vp, vp, vp, vp],
            "dsp_layer_norm_bwd": [vp, i64, i64, vp, vp, vp, vp, ctypes.c_float, vp, vp, vp],
            "dsp_attention_core_lse": [vp, i64, i64, i64, i64, i32, ctypes.c_int, vp, vp, vp, vp],
            "dsp_attention_core_bwd": [vp, i64, i64, i64, i64, i32, ctypes.c_int, vp, vp, vp, vp, vp, vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.dsp_workspace_bytes.argtypes = [P(Shape), ctypes.c_int]
        L.dsp_workspace_bytes.restype = ctypes.c_size_t
        L.dsp_cross_workspace_bytes.argtypes = [P(Shape), ctypes.c_int, i64]
        L.dsp_cross_workspace_bytes.restype = ctypes.c_size_t
        L.dsp_nd_workspace_bytes.argtypes = [P(i64), ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.dsp_nd_workspace_bytes.restype = ctypes.c_size_t
        L.dsp_ulysses_workspace_bytes.argtypes = [P(Shape), ctypes.c_int]
        L.dsp_ulysses_workspace_bytes.restype = ctypes.c_size_t
        L.dsp_train_workspace_bytes.argtypes = [P(Shape), ctypes.c_int]
        L.dsp_train_workspace_bytes.restype = ctypes.c_size_t
        L.dsp_wgrad_workspace_bytes.argtypes = [vp, i64, i64, i64]
        L.dsp_wgrad_workspace_bytes.restype = ctypes.c_size_t
        L.dsp_attention_bwd_workspace_bytes.argtypes = [i64, i64, i32]
        L.dsp_attention_bwd_workspace_bytes.restype = ctypes.c_size_t
        L.dsp_block_prepared_bytes.argtypes = [P(Shape)]
        L.dsp_block_prepared_bytes.restype = ctypes.c_size_t
        L.dsp_status_str.argtypes = [ctypes.c_int]
        L.dsp_status_str.restype = ctypes.c_char_p
        L.dsp_last_error.argtypes = [vp]
        L.dsp_last_error.restype = ctypes.c_char_p
        L.dsp_abi_version.restype = ctypes.c_int
        L.dsp_ctx_launch_count.argtypes = [vp]
        L.dsp_ctx_launch_count.restype = ctypes.c_int64
        _lib = L
    return _lib


def _check(code: int, ctx_handle=None):
    if code != 0:
        msg = lib().dsp_last_error(ctx_handle).decode()
        raise DSPError(code, msg)


def _dtype_code(dt) -> int:
    if dt in (torch.bfloat16, "bf16", DSP_BF16):
        return DSP_BF16
    if dt in (torch.float32, "f32", DSP_F32):
        return DSP_F32
    raise ValueError(f"unsupported dtype {dt}")


def make_shape(B, T, S, C, num_heads, dtype) -> Shape:
    return Shape(int(B), int(T), int(S), int(C), int(num_heads), _dtype_code(dtype))


def _ptr(t) -> int | None:
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch.Tensor")
    if not t.is_cuda:
        raise ValueError("dsp operates on CUDA tensors only (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("dsp needs contiguous tensors")
    return t.data_ptr()


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def workspace_bytes(shape: Shape, world: int) -> int:
    return int(lib().dsp_workspace_bytes(ctypes.byref(shape), int(world)))


def ulysses_workspace_bytes(shape: Shape, world: int) -> int:
    """dsp_ulysses_workspace_bytes: per-rank workspace of the Ulysses-schedule block."""
    return int(lib().dsp_ulysses_workspace_bytes(ctypes.byref(shape), int(world)))


def train_workspace_bytes(shape: Shape, world: int) -> int:
    """dsp_train_workspace_bytes: per-rank workspace of forward_train / backward."""
    return int(lib().dsp_train_workspace_bytes(ctypes.byref(shape), int(world)))


def train_saved_layout(shape: Shape, world: int) -> dict:
    """dsp_train_saved_layout: byte offsets of the saved activations (+ "total")."""
    L = SavedLayout()
    _check(lib().dsp_train_saved_layout(ctypes.byref(shape), int(world), ctypes.byref(L)))
    return {n: int(getattr(L, n)) for n in SAVED_NAMES + ("total",)}


def attention_bwd_workspace_bytes(tok: int, C: int, num_heads: int) -> int:
    return int(lib().dsp_attention_bwd_workspace_bytes(int(tok), int(C), int(num_heads)))


def prepared_bytes(shape: Shape) -> int:
    """Size of the LayerNorm-folded weights buffer of one bf16 block (dsp_block_prepared_bytes)."""
    return int(lib().dsp_block_prepared_bytes(ctypes.byref(shape)))


def switch_volume(shape: Shape, world: int):
    s, r = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().dsp_switch_volume(ctypes.byref(shape), int(world), ctypes.byref(s), ctypes.byref(r)))
    return s.value, r.value


def switch_plan(shape: Shape, world: int, rank: int, from_dim, to_dim) -> SwitchPlan:
    p = SwitchPlan()
    _check(lib().dsp_switch_plan(ctypes.byref(shape), int(world), int(rank), DIMS[from_dim], DIMS[to_dim],
                                 ctypes.byref(p)))
    return p


def cross_workspace_bytes(shape: Shape, world: int, Lc: int) -> int:
    return int(lib().dsp_cross_workspace_bytes(ctypes.byref(shape), int(world), int(Lc)))


def nd_workspace_bytes(dims, dtype, world: int) -> int:
    d = (ctypes.c_int64 * len(dims))(*[int(v) for v in dims])
    return int(lib().dsp_nd_workspace_bytes(d, len(dims), _dtype_code(dtype), int(world)))


def switch_nd_plan(dims, elem_bytes: int, world: int, rank: int, from_dim: int, to_dim: int) -> SwitchNdPlan:
    """dsp_switch_nd_plan (host-only): the byte plan of an N-D switch (dims = global extents, channel last)."""
    p = SwitchNdPlan()
    d = (ctypes.c_int64 * len(dims))(*[int(v) for v in dims])
    _check(lib().dsp_switch_nd_plan(d, len(dims), int(elem_bytes), int(world), int(rank), int(from_dim), int(to_dim),
                                    ctypes.byref(p)))
    return p


def nccl_comm_ptr(pg) -> int:
    """ncclComm_t of an eagerly-initialised ProcessGroupNCCL (init_process_group(..., device_id=...))."""
    backend = pg._get_backend(torch.device("cuda"))
    return int(backend._comm_ptr())


class Context:
    """One dsp context per (process, device, communicator).

    world == 1 needs no process group.  For world > 1 pass the NCCL process group
    (initialised eagerly with device_id so its communicator exists); the context
    borrows its ncclComm_t.  `rank`/`world` may be overridden to build "virtual
    ranks" on one device for the P2P switch tests.
    """

    def __init__(self, pg=None, device=None, rank=None, world=None, comm_ptr=None):
        if not torch.cuda.is_available():
            raise RuntimeError("dsp needs a CUDA device")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   (device.index if isinstance(device, torch.device) else int(device)))
        if pg is not None:
            import torch.distributed as dist
            rank = dist.get_rank(pg) if rank is None else rank
            world = dist.get_world_size(pg) if world is None else world
            if comm_ptr is None and world > 1:
                comm_ptr = nccl_comm_ptr(pg)
        self.rank = 0 if rank is None else int(rank)
        self.world = 1 if world is None else int(world)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib().dsp_ctx_create(comm_ptr, self.rank, self.world, self.device.index, ctypes.byref(h)))
        self.handle = h
        self._ws = None
        self._keep = []

    def close(self):
        if getattr(self, "handle", None):
            lib().dsp_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _call(self, name, *args):
        with torch.cuda.device(self.device):
            _check(getattr(lib(), name)(self.handle, *args), self.handle)

    # ---- resources
    def set_workspace(self, ws: torch.Tensor):
        self._ws = ws
        _check(lib().dsp_ctx_set_workspace(self.handle, _ptr(ws), ws.numel() * ws.element_size()), self.handle)

    def ensure_workspace(self, nbytes: int):
        if self._ws is None or self._ws.numel() < nbytes:
            self.set_workspace(torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device))
        return self._ws

    def set_peer_buffers(self, base_ptrs, signal_ptrs, nbytes: int):
        n = len(base_ptrs)
        B = (ctypes.c_void_p * n)(*base_ptrs)
        S = (ctypes.c_void_p * n)(*signal_ptrs)
        _check(lib().dsp_ctx_set_peer_buffers(self.handle, B, S, int(nbytes)), self.handle)

    def set_barrier_timeout(self, seconds: float):
        """dsp_ctx_set_barrier_timeout: wall-clock bound of a P2P barrier wait (<= 0: forever)."""
        _check(lib().dsp_ctx_set_barrier_timeout(self.handle, float(seconds)), self.handle)

    def set_collective_emulation(self, on: bool = True):
        """dsp_ctx_set_collective_emulation (test infrastructure): NCCL all-to-all / all-gather of this
        virtual rank emulated over the peer mappings (barrier + pull kernel + barrier)."""
        _check(lib().dsp_ctx_set_collective_emulation(self.handle, int(bool(on))), self.handle)

    def check_errors(self):
        """dsp_ctx_check_errors (synchronous): raise DSPError on a timed-out P2P barrier or an
        asynchronous NCCL error of the borrowed communicator."""
        self._call("dsp_ctx_check_errors")

    # ---- instrumentation
    TAPS = {"y1": 0, "y2": 1}

    def set_tap(self, point: str, dst=None):
        """dsp_ctx_set_tap: copy the block's y1 / y2 (S-sharded) into dst on every block call."""
        _check(lib().dsp_ctx_set_tap(self.handle, self.TAPS[point], _ptr(dst),
                                     0 if dst is None else dst.numel() * dst.element_size()), self.handle)

    def set_stage_clocks(self, clocks=None):
        """dsp_ctx_set_stage_clocks: clocks = int64 CUDA tensor [len(STAGES), 2] (reset to
        [max, 0] before each block; read back as ns spans per stage), or None (off)."""
        self._clocks = clocks
        _check(lib().dsp_ctx_set_stage_clocks(self.handle, _ptr(clocks)), self.handle)

    def launch_count(self) -> int:
        return int(lib().dsp_ctx_launch_count(self.handle))

    def set_stage_events(self, events):
        """events: list of 2*len(STAGES) torch.cuda.Event(enable_timing=True) (entries may be None:
        that boundary is not recorded), or None to switch stage events off."""
        if events is None:
            _check(lib().dsp_ctx_set_stage_events(self.handle, None, 0), self.handle)
            self._stage_events = None
            return
        for e in events:
            if e is not None:
                e.record()  # materialise the underlying cudaEvent_t
        arr = (ctypes.c_void_p * len(events))(*[None if e is None else e.cuda_event for e in events])
        self._stage_events = (events, arr)
        _check(lib().dsp_ctx_set_stage_events(self.handle, arr, len(events)), self.handle)

    # ---- layout ops
    def split(self, shape, dim, x_global, x_local, stream=None):
        self._call("dsp_split", ctypes.byref(shape), DIMS[dim], _ptr(x_global), _ptr(x_local), _stream(stream))

    def gather(self, shape, dim, x_local, x_global, stream=None):
        self._call("dsp_gather", ctypes.byref(shape), DIMS[dim], _ptr(x_local), _ptr(x_global), _stream(stream))

    def switch(self, shape, from_dim, to_dim, x_local, y_local, impl="nccl", stream=None):
        self._call("dsp_switch", ctypes.byref(shape), DIMS[from_dim], DIMS[to_dim], _ptr(x_local), _ptr(y_local),
                   IMPLS[impl] if isinstance(impl, str) else int(impl), _stream(stream))

    def switch_pack(self, shape, from_dim, to_dim, x_local, send, stream=None):
        """dsp_switch_pack: x_local -> per-peer chunks [peer][b][t'][s'][c] (NCCL transport, step 1)."""
        self._call("dsp_switch_pack", ctypes.byref(shape), DIMS[from_dim], DIMS[to_dim], _ptr(x_local), _ptr(send),
                   _stream(stream))

    def switch_unpack(self, shape, from_dim, to_dim, recv, y_local, stream=None):
        """dsp_switch_unpack: received chunks [source rank][b][t'][s'][c] -> y_local (step 3)."""
        self._call("dsp_switch_unpack", ctypes.byref(shape), DIMS[from_dim], DIMS[to_dim], _ptr(recv), _ptr(y_local),
                   _stream(stream))

    def gather_unpack(self, shape, dim, gathered, x_global, stream=None):
        """dsp_gather_unpack: all-gathered [N][local] shards -> the global [B,T,S,C] layout."""
        self._call("dsp_gather_unpack", ctypes.byref(shape), DIMS[dim], _ptr(gathered), _ptr(x_global),
                   _stream(stream))

    def switch_nd(self, dims, from_dim: int, to_dim: int, x_local, y_local, impl="nccl", stream=None):
        """dsp_switch_nd: N-D dynamic switch of the global [dims] tensor (channel last) between two dims."""
        d = (ctypes.c_int64 * len(dims))(*[int(v) for v in dims])
        self._call("dsp_switch_nd", d, len(dims), x_local.element_size(), int(from_dim), int(to_dim), _ptr(x_local),
                   _ptr(y_local), IMPLS[impl] if isinstance(impl, str) else int(impl), _stream(stream))

    # ---- N-D block (multi-dimensional transformer; DSP schedule P:93)
    def nd_block_forward(self, dims, num_heads: int, attn_dims, stages, mlp, shard_dim: int, x_local, y_local,
                         impl="nccl", eps: float = 1e-5, stream=None):
        """stages: per attended dim, dict(ln_w, ln_b, w_qkv, w_o); mlp: dict(ln_w, ln_b, w_fc1, w_fc2)."""
        d = (ctypes.c_int64 * len(dims))(*[int(v) for v in dims])
        order = (ctypes.c_int * len(attn_dims))(*[int(k) for k in attn_dims])
        aw = (AttnWeights * len(stages))(*[AttnWeights(*[_ptr(w[n]) for n in ("ln_w", "ln_b", "w_qkv", "w_o")])
                                           for w in stages])
        mw = MlpWeights(*[_ptr(mlp[n]) for n in ("ln_w", "ln_b", "w_fc1", "w_fc2")])
        self._call("dsp_nd_block_forward", d, len(dims), int(num_heads), _dtype_code(x_local.dtype), len(stages),
                   order, aw, ctypes.byref(mw), ctypes.c_float(eps), int(shard_dim), _ptr(x_local), _ptr(y_local),
                   IMPLS[impl] if isinstance(impl, str) else int(impl), _stream(stream))

    # ---- compute
    def spatial_attn(self, shape, h, w_qkv, w_o, residual, out, stream=None):
        self._call("dsp_spatial_attn", ctypes.byref(shape), _ptr(h), _ptr(w_qkv), _ptr(w_o), _ptr(residual),
                   _ptr(out), _stream(stream))

    def cross_attn(self, shape, h, ctx_tokens, w_q, w_kv, w_o, residual, out, stream=None):
        """dsp_cross_attn: out = residual + CA(h, ctx_tokens) (ctx_tokens [B, Lc, C])."""
        Lc = ctx_tokens.numel() // (shape.B * shape.C)
        self._call("dsp_cross_attn", ctypes.byref(shape), _ptr(h), _ptr(ctx_tokens), int(Lc), _ptr(w_q), _ptr(w_kv),
                   _ptr(w_o), _ptr(residual), _ptr(out), _stream(stream))

    def temporal_attn(self, shape, h, w_qkv, w_o, residual, out, stream=None):
        self._call("dsp_temporal_attn", ctypes.byref(shape), _ptr(h), _ptr(w_qkv), _ptr(w_o), _ptr(residual),
                   _ptr(out), _stream(stream))

    # ---- training path (include/dsp_train.h)
    def block_forward_train(self, shape, W: dict, x_local, y_local, saved, impl="nccl", stream=None):
        """dsp_st_block_forward_train: the block forward, keeping its activations in `saved` (uint8 CUDA
        tensor of train_saved_layout(...)["total"] bytes)."""
        bw = self.block_weights(W)
        self._call("dsp_st_block_forward_train", ctypes.byref(shape), ctypes.byref(bw), _ptr(x_local), _ptr(y_local),
                   _ptr(saved), IMPLS[impl] if isinstance(impl, str) else int(impl), _stream(stream))

    def block_backward(self, shape, W: dict, saved, x_local, dy_local, dx_local, grads: dict, impl="nccl",
                       stream=None):
        """dsp_st_block_backward: dx_local and grads[name] += dW (fp32 CUDA tensors, GRAD_NAMES)."""
        bw = self.block_weights(W)
        g = BlockGrads(*[_ptr(grads[n]) for n in GRAD_NAMES])
        self._call("dsp_st_block_backward", ctypes.byref(shape), ctypes.byref(bw), _ptr(saved), _ptr(x_local),
                   _ptr(dy_local), _ptr(dx_local), ctypes.byref(g), IMPLS[impl] if isinstance(impl, str) else int(impl),
                   _stream(stream))

    def grads_reduce(self, buf, zero_shard: bool = False, out=None, stream=None):
        """dsp_grads_reduce: NCCL all-reduce (or ZeRO reduce-scatter into out) of fp32 gradients."""
        self._call("dsp_grads_reduce", _ptr(buf), buf.numel(), int(bool(zero_shard)), _ptr(out), _stream(stream))

    def linear_dgrad(self, dY, W, dX, u=None, stream=None):
        """dsp_linear_dgrad: dX[M, K] = dY[M, N] W[N, K] (* gelu'(u) if u is given)."""
        N = W.shape[0]
        M = dY.numel() // N
        self._call("dsp_linear_dgrad", M, N, W.shape[1], _ptr(dY), _ptr(W), _ptr(u), _ptr(dX), _stream(stream))

    def linear_wgrad(self, dY, X, dW, accumulate=False, stream=None):
        """dsp_linear_wgrad: dW[N, K] (+)= dY[M, N]^T X[M, K] in fp32 (needs dsp_wgrad_workspace_bytes)."""
        N, K = dW.shape
        M = dY.numel() // N
        self.ensure_workspace(int(lib().dsp_wgrad_workspace_bytes(self.handle, M, N, K)))
        self._call("dsp_linear_wgrad", M, N, K, _ptr(dY), _ptr(X), _ptr(dW), int(bool(accumulate)), _stream(stream))

    def linear_gelu_aux(self, A, W, G, U, stream=None):
        """dsp_linear_gelu_aux: G = gelu_tanh(A W^T), U = A W^T."""
        N, K = W.shape
        self._call("dsp_linear_gelu_aux", A.numel() // K, N, K, _ptr(A), _ptr(W), _ptr(G), _ptr(U), _stream(stream))

    def layer_norm_bwd(self, x, gamma, dh, dres, dx, dgamma_dbeta, eps=1e-5, stream=None):
        """dsp_layer_norm_bwd: dx = dres + LN^T dh; dgamma_dbeta[2C] += (sum dh xhat, sum dh)."""
        C = x.shape[-1]
        self._call("dsp_layer_norm_bwd", x.numel() // C, C, _ptr(x), _ptr(gamma), _ptr(dh), _ptr(dres),
                   ctypes.c_float(eps), _ptr(dx), _ptr(dgamma_dbeta), _stream(stream))

    def attention_core_lse(self, B, T_loc, S_loc, C, num_heads, dim, qkv, o, lse, stream=None):
        self._call("dsp_attention_core_lse", int(B), int(T_loc), int(S_loc), int(C), int(num_heads), DIMS[dim],
                   _ptr(qkv), _ptr(o), _ptr(lse), _stream(stream))

    def attention_core_bwd(self, B, T_loc, S_loc, C, num_heads, dim, qkv, o, dout, lse, dqkv, stream=None):
        self.ensure_workspace(attention_bwd_workspace_bytes(B * T_loc * S_loc, C, num_heads))
        self._call("dsp_attention_core_bwd", int(B), int(T_loc), int(S_loc), int(C), int(num_heads), DIMS[dim],
                   _ptr(qkv), _ptr(o), _ptr(dout), _ptr(lse), _ptr(dqkv), _stream(stream))

    @staticmethod
    def block_weights(W: dict, eps: float = 1e-5) -> BlockWeights:
        """W: the 12 weight tensors by name, plus optionally "prepared" (from prepare_block), the
        cross stage (CROSS_NAMES + "ctx_tokens" [B, Lc, C]), the Latte pair (LATTE_NAMES) and the
        temporal positional embedding "pe_t" [T, C]."""
        prep = W.get("prepared")
        cross = [None] * 5 + [None, 0]
        if W.get("ln_c_w") is not None:
            ctxt = W["ctx_tokens"]
            cross = [_ptr(W[n]) for n in CROSS_NAMES] + [_ptr(ctxt), int(ctxt.shape[-2])]
        latte = [_ptr(W[n]) if W.get(n) is not None else None for n in LATTE_NAMES]
        pe = W.get("pe_t")
        return BlockWeights(*[_ptr(W[n]) for n in WEIGHT_NAMES], ctypes.c_float(eps),
                            None if prep is None else _ptr(prep), *cross, *latte, None if pe is None else _ptr(pe))

    def adaln_fold(self, shape, W: dict, mod: torch.Tensor, stream=None) -> dict:
        """dsp_adaln_fold (R36, B = 1): returns a copy of W whose LayerNorm parameters and output
        projections carry sample 0's adaLN-Zero modulation; mod: f32 CUDA tensor [4, 3, C] rows
        (shift, scale, gate) for ADALN_SUBLAYERS (the spatial-MLP row is read only with a Latte pair)."""
        out = {k: v for k, v in W.items() if k != "prepared"}
        names = ["ln1_w", "ln1_b", "w_o_s", "ln2_w", "ln2_b", "w_o_t", "ln3_w", "ln3_b", "w_fc2"]
        if W.get("w_fc1_s") is not None:
            names += ["ln_m_w", "ln_m_b", "w_fc2_s"]
        for n in names:
            out[n] = torch.empty_like(W[n])
        bw_in = self.block_weights({k: v for k, v in W.items() if k != "prepared"})
        bw_out = self.block_weights(out)
        self._call("dsp_adaln_fold", ctypes.byref(shape), ctypes.byref(bw_in), _ptr(mod.contiguous()),
                   ctypes.byref(bw_out), _stream(stream))
        return out

    def prepare_block(self, shape, W: dict, prepared=None, stream=None) -> torch.Tensor:
        """dsp_st_block_prepare: fold the three LayerNorms into their GEMMs' weights once.
        Returns the prepared buffer; pass it as W["prepared"] to st_block_forward."""
        if prepared is None:  # f32 shapes: 0 bytes -> the C call reports DSP_ERR_UNSUPPORTED
            prepared = torch.empty(max(prepared_bytes(shape), 256), dtype=torch.uint8, device=self.device)
        bw = self.block_weights({k: v for k, v in W.items() if k != "prepared"})  # incl. the cross stage
        self._call("dsp_st_block_prepare", ctypes.byref(shape), ctypes.byref(bw), _ptr(prepared),
                   prepared.numel() * prepared.element_size(), _stream(stream))
        return prepared

    def st_block_forward(self, shape, weights, x_local, y_local, impl="nccl", stream=None):
        bw = weights if isinstance(weights, BlockWeights) else self.block_weights(weights)
        self._call("dsp_st_block_forward", ctypes.byref(shape), ctypes.byref(bw), _ptr(x_local), _ptr(y_local),
                   IMPLS[impl] if isinstance(impl, str) else int(impl), _stream(stream))

    def st_block_forward_ulysses(self, shape, weights, x_local, y_local, impl="nccl", stream=None):
        """dsp_st_block_forward_ulysses: the same block under DeepSpeed-Ulysses (4 all-to-alls per
        attention stage; T-sharded in and out)."""
        bw = weights if isinstance(weights, BlockWeights) else self.block_weights(weights)
        self._call("dsp_st_block_forward_ulysses", ctypes.byref(shape), ctypes.byref(bw), _ptr(x_local),
                   _ptr(y_local), IMPLS[impl] if isinstance(impl, str) else int(impl), _stream(stream))

    def st_model_forward(self, shape, layers, x_local, y_local, impl="nccl", stream=None):
        """dsp_st_model_forward: layers = list of per-layer weights (dicts or BlockWeights)."""
        bws = [w if isinstance(w, BlockWeights) else self.block_weights(w) for w in layers]
        arr = (ctypes.POINTER(BlockWeights) * len(bws))(*[ctypes.pointer(b) for b in bws])
        self._keep_model = (bws, arr)
        self._call("dsp_st_model_forward", ctypes.byref(shape), arr, len(bws), _ptr(x_local), _ptr(y_local),
                   IMPLS[impl] if isinstance(impl, str) else int(impl), _stream(stream))

    def st_block_forward_host(self, shape, weights, x_host: torch.Tensor, y_host: torch.Tensor, x_dev, y_dev,
                              impl="nccl", stream=None):
        bw = weights if isinstance(weights, BlockWeights) else self.block_weights(weights)
        for t in (x_host, y_host):
            if t.is_cuda or not t.is_contiguous():
                raise ValueError("host buffers must be contiguous CPU tensors (pinned recommended)")
        self._call("dsp_st_block_forward_host", ctypes.byref(shape), ctypes.byref(bw), x_host.data_ptr(),
                   y_host.data_ptr(), _ptr(x_dev), _ptr(y_dev), IMPLS[impl] if isinstance(impl, str) else int(impl),
                   _stream(stream))

    def st_block_forward_host_pipelined(self, shape, weights, x_hosts, y_hosts, x_devs, y_devs, impl="nccl",
                                        stream=None):
        """dsp_st_block_forward_host_pipelined: len(x_hosts) independent blocks with their H2D / D2H
        copies overlapped across steps (x_devs, y_devs: two device staging buffers each)."""
        bw = weights if isinstance(weights, BlockWeights) else self.block_weights(weights)
        n = len(x_hosts)
        if len(y_hosts) != n or len(x_devs) != 2 or len(y_devs) != 2:
            raise ValueError("need n host inputs, n host outputs, 2 + 2 device staging buffers")
        for t in list(x_hosts) + list(y_hosts):
            if t.is_cuda or not t.is_contiguous():
                raise ValueError("host buffers must be contiguous CPU tensors (pinned recommended)")
        arr = lambda ptrs: (ctypes.c_void_p * max(len(ptrs), 1))(*ptrs)
        self._call("dsp_st_block_forward_host_pipelined", ctypes.byref(shape), ctypes.byref(bw), n,
                   arr([t.data_ptr() for t in x_hosts]), arr([t.data_ptr() for t in y_hosts]),
                   arr([_ptr(t) for t in x_devs]), arr([_ptr(t) for t in y_devs]),
                   IMPLS[impl] if isinstance(impl, str) else int(impl), _stream(stream))

    def layer_norm(self, x, gamma, beta, eps, y, stream=None):
        rows, C = x.numel() // x.shape[-1], x.shape[-1]
        self._call("dsp_layer_norm", _dtype_code(x.dtype), rows, C, _ptr(x), _ptr(gamma), _ptr(beta),
                   ctypes.c_float(eps), _ptr(y), _stream(stream))

    def linear(self, A, W, D, R=None, epi=DSP_EPI_NONE, stream=None):
        M, K = A.numel() // A.shape[-1], A.shape[-1]
        N = W.shape[0]
        self._call("dsp_linear", _dtype_code(A.dtype), M, N, K, _ptr(A), _ptr(W), _ptr(R), int(epi), _ptr(D),
                   _stream(stream))

    def attention_core(self, B, T_loc, S_loc, C, num_heads, dim, qkv, o, stream=None):
        self._call("dsp_attention_core", _dtype_code(qkv.dtype), B, T_loc, S_loc, C, num_heads, DIMS[dim],
                   _ptr(qkv), _ptr(o), _stream(stream))
