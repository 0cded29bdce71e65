"""B200-native pruned RNN-T loss hot path (arXiv 2206.13236) — Python binding.

Thin ctypes binding over ``librnnt_b200.so`` (the C-ABI of ``include/rnnt.h``):
argument marshalling only, every step of the path runs in the library's sm_100a
kernels.  PyTorch supplies device memory and streams.  There is no CPU fallback:
if the shared library is missing or a tensor is not on a CUDA device, the calls
raise.

Two layers:
  * ``rnnt_simple_loss``, ``rnnt_get_ranges``, ``rnnt_prune``, ``rnnt_pruned_loss``,
    ``rnnt_workspace_bytes`` — same names and argument order as the C-ABI, taking
    torch tensors (or None for nullable pointers).
  * ``simple_loss``, ``get_ranges``, ``prune``, ``pruned_loss`` and ``step`` —
    conveniences that allocate outputs with ``torch.empty`` and call the above.
"""
from __future__ import annotations

import ctypes
import os
import re

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librnnt_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "rnnt.h")

RNNT_OK = 0
STATUS_INFEASIBLE = 1
STATUS_NONFINITE = 2
STATUS_BAD_SYMBOL = 4
STATUS_UNDERFLOW = 8
STATUS_BAD_BOUNDARY = 16

EXCHANGE_STORE = 0      # rnnt_exchange_mode_t (include/rnnt.h)
EXCHANGE_RED = 1
EXCHANGE_MULTIMEM = 2


class Dims(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("T", ctypes.c_int32), ("U", ctypes.c_int32),
                ("V", ctypes.c_int32), ("J", ctypes.c_int32), ("S", ctypes.c_int32)]


class RNNTError(RuntimeError):
    pass


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the C-ABI library (raises if it is not built).  RNNT_LIB overrides the path (A/B
    comparisons of two builds of the same library in tools/)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("RNNT_LIB", path)
    if not os.path.exists(path):
        raise RNNTError(f"{path} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, I32, F, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_float, ctypes.c_size_t
    DP = ctypes.POINTER(Dims)
    lib.rnnt_workspace_bytes.argtypes = [DP]
    lib.rnnt_workspace_bytes.restype = SZ
    lib.rnnt_status_string.argtypes = [I32]
    lib.rnnt_status_string.restype = ctypes.c_char_p
    lib.rnnt_version.argtypes = []
    lib.rnnt_version.restype = ctypes.c_char_p
    lib.rnnt_last_cuda_error.argtypes = []
    lib.rnnt_last_cuda_error.restype = ctypes.c_char_p
    lib.rnnt_simple_loss.argtypes = [P, P, P, P, DP, F, P, P, P, P, P, P, P, SZ, P]
    lib.rnnt_simple_loss.restype = I32
    lib.rnnt_simple_loss_backward.argtypes = [P, P, P, P, P, P, DP, F, P, P, P, SZ, P]
    lib.rnnt_simple_loss_backward.restype = I32
    lib.rnnt_full_workspace_bytes.argtypes = [DP]
    lib.rnnt_full_workspace_bytes.restype = SZ
    lib.rnnt_full_loss.argtypes = [P, P, P, P, P, P, DP, F, P, P, P, P, P, P, P, SZ, P]
    lib.rnnt_full_loss.restype = I32
    lib.rnnt_simple_loss_smoothed.argtypes = [P, P, P, P, DP, F, F, F, P, P, P, P, P, P, P, SZ, P]
    lib.rnnt_simple_loss_smoothed.restype = I32
    lib.rnnt_simple_loss_smoothed_backward.argtypes = [P, P, P, P, P, P, DP, F, F, F, P, P, P, SZ, P]
    lib.rnnt_simple_loss_smoothed_backward.restype = I32
    lib.rnnt_get_ranges.argtypes = [P, P, P, DP, P, P, P]
    lib.rnnt_get_ranges.restype = I32
    lib.rnnt_prune.argtypes = [P, P, P, P, DP, P, P]
    lib.rnnt_prune.restype = I32
    lib.rnnt_pruned_loss.argtypes = [P, P, P, P, P, P, DP, F, P, P, P, P, P, P, P, SZ, P]
    lib.rnnt_pruned_loss.restype = I32
    lib.rnnt_pruned_loss_forward.argtypes = [P, P, P, P, P, P, DP, F, P, P, P, SZ, P]
    lib.rnnt_pruned_loss_forward.restype = I32
    lib.rnnt_pruned_loss_prepare.argtypes = [P, P, P, DP, P, F, P, SZ, P]
    lib.rnnt_pruned_loss_prepare.restype = I32
    lib.rnnt_pruned_loss_forward_prepared.argtypes = lib.rnnt_pruned_loss_forward.argtypes
    lib.rnnt_pruned_loss_forward_prepared.restype = I32
    lib.rnnt_pruned_loss_backward_input.argtypes = [P, P, P, P, DP, P, P, P, SZ, P]
    lib.rnnt_pruned_loss_backward_input.restype = I32
    lib.rnnt_pruned_loss_backward_weight.argtypes = [P, DP, P, P, P, SZ, P]
    lib.rnnt_pruned_loss_backward_weight.restype = I32
    lib.rnnt_pruned_loss_backward_weight_exchange.argtypes = [P, DP, I32, P, P, P, SZ, P]
    lib.rnnt_pruned_loss_backward_weight_exchange.restype = I32
    lib.rnnt_exchange_sum.argtypes = [P, I32, ctypes.c_int64, I32, P, P]
    lib.rnnt_exchange_sum.restype = I32
    lib.rnnt_loss_sums.argtypes = [P, P, P, I32, F, F, I32, P, P]
    lib.rnnt_loss_sums.restype = I32
    lib.rnnt_launch_count.argtypes = []
    lib.rnnt_launch_count.restype = ctypes.c_uint64
    lib.rnnt_pruned_backward_mode.argtypes = [ctypes.POINTER(Dims), P, ctypes.c_size_t, ctypes.POINTER(I32), P]
    lib.rnnt_pruned_backward_mode.restype = I32
    lib.rnnt_kernel_count.argtypes = []
    lib.rnnt_kernel_count.restype = I32
    lib.rnnt_kernel_name.argtypes = [I32]
    lib.rnnt_kernel_name.restype = ctypes.c_char_p
    lib.rnnt_profile_kernel.argtypes = [I32, P, P]
    lib.rnnt_profile_kernel.restype = I32
    _lib = lib
    return lib


def header_functions(path: str = HEADER_PATH) -> list[str]:
    """Names of the functions declared in include/rnnt.h."""
    src = open(path).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rnnt_[a-z_]+)\s*\(", src)))


def _ptr(t):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch.Tensor")
    if not t.is_cuda:
        raise RNNTError("tensor must be on a CUDA device (no CPU fallback)")
    if not t.is_contiguous():
        raise RNNTError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _check(rc: int, what: str):
    if rc != RNNT_OK:
        lib = load_library()
        msg = lib.rnnt_status_string(rc).decode()
        if msg == "RNNT_ERR_CUDA":
            msg += " (" + lib.rnnt_last_cuda_error().decode() + ")"
        raise RNNTError(f"{what} failed: {msg}")


def make_dims(N, T, U, V, J, S) -> Dims:
    return Dims(int(N), int(T), int(U), int(V), int(J), int(S))


# ----------------------------------------------------------------- C-ABI mirror
def rnnt_workspace_bytes(dims: Dims) -> int:
    return int(load_library().rnnt_workspace_bytes(ctypes.byref(dims)))


def rnnt_version() -> str:
    return load_library().rnnt_version().decode()


def rnnt_launch_count() -> int:
    return int(load_library().rnnt_launch_count())


def rnnt_pruned_backward_mode(dims, workspace, stream=None) -> bool:
    """True if the last rnnt_pruned_loss_forward in `workspace` selected the plain joiner backward
    (one P~ offset per row; include/rnnt.h, D20).  Synchronises the stream."""
    out = ctypes.c_int32(0)
    rc = load_library().rnnt_pruned_backward_mode(ctypes.byref(dims), _ptr(workspace), workspace.numel() *
                                                  workspace.element_size(), ctypes.byref(out), _stream(stream))
    _check(rc, "rnnt_pruned_backward_mode")
    return bool(out.value)


def kernel_ids() -> dict:
    """{kernel name: id} of the library's launch sites."""
    lib = load_library()
    return {lib.rnnt_kernel_name(i).decode(): i for i in range(1, lib.rnnt_kernel_count())}


def rnnt_profile_kernel(kernel_id: int, start_event=None, stop_event=None):
    """Bracket every later launch of ``kernel_id`` (from this thread) with the two
    torch.cuda.Event objects (recorded on the launch stream); kernel_id 0 disarms."""
    s = ctypes.c_void_p(start_event.cuda_event) if start_event is not None else None
    e = ctypes.c_void_p(stop_event.cuda_event) if stop_event is not None else None
    _check(load_library().rnnt_profile_kernel(int(kernel_id), s, e), "rnnt_profile_kernel")


def rnnt_simple_loss(am, lm, symbols, boundary, dims, grad_scale, loss, px_grad, py_grad, am_grad,
                     lm_grad, status, workspace, stream=None):
    rc = load_library().rnnt_simple_loss(
        _ptr(am), _ptr(lm), _ptr(symbols), _ptr(boundary), ctypes.byref(dims), float(grad_scale),
        _ptr(loss), _ptr(px_grad), _ptr(py_grad), _ptr(am_grad), _ptr(lm_grad), _ptr(status),
        _ptr(workspace), workspace.numel() * workspace.element_size(), _stream(stream))
    _check(rc, "rnnt_simple_loss")


def rnnt_simple_loss_backward(am, lm, px_grad, py_grad, symbols, boundary, dims, grad_scale, am_grad, lm_grad,
                              workspace, stream=None):
    rc = load_library().rnnt_simple_loss_backward(
        _ptr(am), _ptr(lm), _ptr(px_grad), _ptr(py_grad), _ptr(symbols), _ptr(boundary), ctypes.byref(dims),
        float(grad_scale), _ptr(am_grad), _ptr(lm_grad), _ptr(workspace), workspace.numel() * workspace.element_size(),
        _stream(stream))
    _check(rc, "rnnt_simple_loss_backward")


def rnnt_simple_loss_smoothed(am, lm, symbols, boundary, dims, lm_only_scale, am_only_scale, grad_scale, loss,
                              px_grad, py_grad, am_grad, lm_grad, status, workspace, stream=None):
    rc = load_library().rnnt_simple_loss_smoothed(
        _ptr(am), _ptr(lm), _ptr(symbols), _ptr(boundary), ctypes.byref(dims), float(lm_only_scale),
        float(am_only_scale), float(grad_scale), _ptr(loss), _ptr(px_grad), _ptr(py_grad), _ptr(am_grad),
        _ptr(lm_grad), _ptr(status), _ptr(workspace), workspace.numel() * workspace.element_size(), _stream(stream))
    _check(rc, "rnnt_simple_loss_smoothed")


def rnnt_simple_loss_smoothed_backward(am, lm, px_grad, py_grad, symbols, boundary, dims, lm_only_scale, am_only_scale,
                                       grad_scale, am_grad, lm_grad, workspace, stream=None):
    rc = load_library().rnnt_simple_loss_smoothed_backward(
        _ptr(am), _ptr(lm), _ptr(px_grad), _ptr(py_grad), _ptr(symbols), _ptr(boundary), ctypes.byref(dims),
        float(lm_only_scale), float(am_only_scale), float(grad_scale), _ptr(am_grad), _ptr(lm_grad), _ptr(workspace),
        workspace.numel() * workspace.element_size(), _stream(stream))
    _check(rc, "rnnt_simple_loss_smoothed_backward")


def rnnt_full_workspace_bytes(dims) -> int:
    return int(load_library().rnnt_full_workspace_bytes(ctypes.byref(dims)))


def rnnt_full_loss(enc_proj, dec_proj, w_out, b_out, symbols, boundary, dims, grad_scale, loss, d_enc, d_dec, d_w,
                   d_b, status, workspace, stream=None):
    rc = load_library().rnnt_full_loss(
        _ptr(enc_proj), _ptr(dec_proj), _ptr(w_out), _ptr(b_out), _ptr(symbols), _ptr(boundary), ctypes.byref(dims),
        float(grad_scale), _ptr(loss), _ptr(d_enc), _ptr(d_dec), _ptr(d_w), _ptr(d_b), _ptr(status), _ptr(workspace),
        workspace.numel() * workspace.element_size(), _stream(stream))
    _check(rc, "rnnt_full_loss")


def full_loss(enc_proj, dec_proj, w_out, b_out, symbols, boundary, grad_scale=1.0, stream=None):
    """The full (unpruned) loss with the same joiner: returns a dict of device
    tensors loss, d_enc, d_dec, d_w, d_b, status (allocates its own workspace)."""
    N, T, J = enc_proj.shape
    U = dec_proj.shape[1] - 1
    V = w_out.shape[0]
    dims = make_dims(N, T, U, V, J, 1)
    dev = enc_proj.device
    f32 = dict(dtype=torch.float32, device=dev)
    o = dict(loss=torch.empty(N, **f32), d_enc=torch.empty(N, T, J, **f32), d_dec=torch.empty(N, U + 1, J, **f32),
             d_w=torch.empty(V, J, **f32), d_b=torch.empty(V, **f32),
             status=torch.zeros(N, dtype=torch.int32, device=dev))
    nbytes = rnnt_full_workspace_bytes(dims)
    if nbytes == 0:
        raise RNNTError("invalid dims for rnnt_full_loss")
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    rnnt_full_loss(enc_proj, dec_proj, w_out, b_out, symbols, boundary, dims, grad_scale, o["loss"], o["d_enc"],
                   o["d_dec"], o["d_w"], o["d_b"], o["status"], ws, stream)
    return o


def rnnt_get_ranges(px_grad, py_grad, boundary, dims, ranges, status, stream=None):
    rc = load_library().rnnt_get_ranges(_ptr(px_grad), _ptr(py_grad), _ptr(boundary), ctypes.byref(dims),
                                        _ptr(ranges), _ptr(status), _stream(stream))
    _check(rc, "rnnt_get_ranges")


def rnnt_prune(enc_proj, dec_proj, ranges, boundary, dims, h, stream=None):
    rc = load_library().rnnt_prune(_ptr(enc_proj), _ptr(dec_proj), _ptr(ranges), _ptr(boundary),
                                   ctypes.byref(dims), _ptr(h), _stream(stream))
    _check(rc, "rnnt_prune")


def rnnt_pruned_loss(h, w_out, b_out, symbols, ranges, boundary, dims, grad_scale, loss, d_enc, d_dec,
                     d_w, d_b, status, workspace, stream=None):
    rc = load_library().rnnt_pruned_loss(
        _ptr(h), _ptr(w_out), _ptr(b_out), _ptr(symbols), _ptr(ranges), _ptr(boundary),
        ctypes.byref(dims), float(grad_scale), _ptr(loss), _ptr(d_enc), _ptr(d_dec), _ptr(d_w),
        _ptr(d_b), _ptr(status), _ptr(workspace), workspace.numel() * workspace.element_size(),
        _stream(stream))
    _check(rc, "rnnt_pruned_loss")


def rnnt_pruned_loss_forward(h, w_out, b_out, symbols, ranges, boundary, dims, grad_scale, loss, status, workspace,
                             stream=None):
    rc = load_library().rnnt_pruned_loss_forward(
        _ptr(h), _ptr(w_out), _ptr(b_out), _ptr(symbols), _ptr(ranges), _ptr(boundary), ctypes.byref(dims),
        float(grad_scale), _ptr(loss), _ptr(status), _ptr(workspace), workspace.numel() * workspace.element_size(),
        _stream(stream))
    _check(rc, "rnnt_pruned_loss_forward")


def rnnt_pruned_loss_prepare(ranges, symbols, boundary, dims, b_out, grad_scale, workspace, stream=None):
    rc = load_library().rnnt_pruned_loss_prepare(
        _ptr(ranges), _ptr(symbols), _ptr(boundary), ctypes.byref(dims), _ptr(b_out), float(grad_scale),
        _ptr(workspace), workspace.numel() * workspace.element_size(), _stream(stream))
    _check(rc, "rnnt_pruned_loss_prepare")


def rnnt_pruned_loss_forward_prepared(h, w_out, b_out, symbols, ranges, boundary, dims, grad_scale, loss, status,
                                      workspace, stream=None):
    rc = load_library().rnnt_pruned_loss_forward_prepared(
        _ptr(h), _ptr(w_out), _ptr(b_out), _ptr(symbols), _ptr(ranges), _ptr(boundary), ctypes.byref(dims),
        float(grad_scale), _ptr(loss), _ptr(status), _ptr(workspace), workspace.numel() * workspace.element_size(),
        _stream(stream))
    _check(rc, "rnnt_pruned_loss_forward_prepared")


def rnnt_pruned_loss_backward_input(h, w_out, ranges, boundary, dims, d_enc, d_dec, workspace, stream=None):
    rc = load_library().rnnt_pruned_loss_backward_input(
        _ptr(h), _ptr(w_out), _ptr(ranges), _ptr(boundary), ctypes.byref(dims), _ptr(d_enc), _ptr(d_dec),
        _ptr(workspace), workspace.numel() * workspace.element_size(), _stream(stream))
    _check(rc, "rnnt_pruned_loss_backward_input")


def rnnt_pruned_loss_backward_weight(h, dims, d_w, d_b, workspace, stream=None):
    rc = load_library().rnnt_pruned_loss_backward_weight(
        _ptr(h), ctypes.byref(dims), _ptr(d_w), _ptr(d_b), _ptr(workspace), workspace.numel() * workspace.element_size(),
        _stream(stream))
    _check(rc, "rnnt_pruned_loss_backward_weight")


def _addr(x):
    """A device pointer: a CUDA tensor, or a raw integer address (e.g. a multicast address)."""
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    return _ptr(x)


def rnnt_pruned_loss_backward_weight_exchange(h, dims, mode, d_w, d_b, workspace, stream=None):
    rc = load_library().rnnt_pruned_loss_backward_weight_exchange(
        _ptr(h), ctypes.byref(dims), int(mode), _addr(d_w), _addr(d_b), _ptr(workspace),
        workspace.numel() * workspace.element_size(), _stream(stream))
    _check(rc, "rnnt_pruned_loss_backward_weight_exchange")


def rnnt_exchange_sum(parts, nparts, M, mode, out, stream=None):
    rc = load_library().rnnt_exchange_sum(_ptr(parts), int(nparts), int(M), int(mode), _addr(out), _stream(stream))
    _check(rc, "rnnt_exchange_sum")


def rnnt_loss_sums(loss_simple, loss_pruned, status, N, simple_scale, pruned_scale, mode, out, stream=None):
    rc = load_library().rnnt_loss_sums(_ptr(loss_simple), _ptr(loss_pruned), _ptr(status), int(N),
                                       float(simple_scale), float(pruned_scale), int(mode), _addr(out),
                                       _stream(stream))
    _check(rc, "rnnt_loss_sums")


# ----------------------------------------------------------------- conveniences
class Workspace:
    """Caches one device workspace per (device, size)."""

    def __init__(self):
        self.buf = None

    def get(self, dims: Dims, device) -> torch.Tensor:
        need = rnnt_workspace_bytes(dims)
        if need == 0:
            raise RNNTError("invalid dims")
        if self.buf is None or self.buf.numel() < need or self.buf.device != torch.device(device):
            self.buf = torch.empty(need, dtype=torch.uint8, device=device)
        return self.buf


_WS = Workspace()


def dims_of(am, lm, w_out, S) -> Dims:
    N, T, V = am.shape
    U = lm.shape[1] - 1
    J = w_out.shape[1]
    return make_dims(N, T, U, V, J, S)


_SIDE = {}


# A/B switch: RNNT_SIMPLE_BWD=late launches the am/lm gradients (side stream) after the pruned forward, so
# they overlap the joiner backward instead of the bounds / gather / joiner forward chain.
_SIMPLE_BWD_LATE = os.environ.get("RNNT_SIMPLE_BWD", "early") == "late"


# The weight-gradient side stream (which = 1) runs at CUDA priority RNNT_DW_PRIO (0 lowest .. -5; default -2):
# above the am / lm gradient stream (which = 0, lowest), below the critical stream.  At the lowest priority its
# kernels queued behind the am-gradient GEMM's pending blocks and d_w -- the last kernel of the step at c3 / c4 --
# started only once that GEMM had drained (c3 1.113 -> 1.089 ms, c4 6.81 -> 6.63 ms, c5 unchanged).
_DW_PRIO = int(os.environ.get("RNNT_DW_PRIO", "-2"))


def _side_stream(device, which=0, lane=0):
    key = (torch.device(device).index, which, lane)
    if key not in _SIDE:
        lo, hi = torch.cuda.Stream.priority_range()
        prio = max(hi, min(lo, _DW_PRIO)) if which == 1 else lo
        _SIDE[key] = torch.cuda.Stream(device=device, priority=prio)   # lowest priority: fills gaps
    return _SIDE[key]


_CRIT = {}


_PREP_LANE = 1000   # critical_stream lanes of the prepare call (lane + 1000: never a sub-batch lane)
# A/B switch: RNNT_SPLIT_PREP=1 runs rnnt_pruned_loss_prepare on its own stream concurrently with the gather
# (the rowinfo launch leaves the chain, but the joiner forward then shares its SMs with the lm gradient)
_SPLIT_PREP = os.environ.get("RNNT_SPLIT_PREP", "0") == "1"   # measured: no change at c5 (0.425 either way)


def critical_stream(device=None, lane=0):
    """A high-priority stream for the step's critical path: with the side streams at the lowest
    priority the block scheduler hands idle SMs (e.g. during the latency-bound recursions) to the
    side-stream GEMMs without delaying the critical-path kernels.  ``lane`` > 0: the critical
    stream of sub-batch ``lane`` of a grouped step."""
    idx = torch.device(device if device is not None else "cuda").index
    idx = torch.cuda.current_device() if idx is None else idx
    if (idx, lane) not in _CRIT:
        lo, hi = torch.cuda.Stream.priority_range()
        _CRIT[(idx, lane)] = torch.cuda.Stream(device=idx, priority=hi)
    return _CRIT[(idx, lane)]


def step(am, lm, symbols, boundary, enc_proj, dec_proj, w_out, b_out, S, simple_scale=0.5,
         pruned_scale=1.0, status=None, workspace=None, out=None, stream=None, overlap=True,
         lm_only_scale=0.0, am_only_scale=0.0, grad_hook=None, exchange=None, lane=0, groups=1):
    """One fwd+bwd of the whole hot path: simple loss and its
    gradients, bounds, gather, pruned loss and joiner gradients.  Returns a dict of
    device tensors; ``out`` may supply preallocated outputs (same keys).

    ``lm_only_scale`` / ``am_only_scale`` select the smoothed trivial joiner (Eq. 11-15) for the
    simple stage (0, 0: the plain trivial joiner).  With ``overlap`` the am/lm gradients
    (rnnt_simple_loss[_smoothed]_backward) run on a side stream concurrently with the pruned stage,
    joined back into ``stream`` before returning.

    ``grad_hook()`` (e.g. the data-parallel all_reduce of d_w / d_b / loss sums) is called once both
    losses and d_w / d_b are final: with ``overlap`` on the d_w stream right after the weight
    gradient, so the collective overlaps the input-gradient kernels; otherwise at the end.

    ``exchange`` (a ``dist.GradBuffer``): the data-parallel exchange.  d_w / d_b are delivered into
    its flat buffer by the library (plain stores + NCCL all_reduce, NVLS multimem adds, or local
    adds), the masked batch-loss sums (rnnt_loss_sums) into its tail, and ``out["d_w"]`` /
    ``out["d_b"]`` are views of it; the reduction overlaps the input-gradient kernels.

    ``groups`` > 1: the batch is cut into that many contiguous sub-batches of utterances whose
    whole chains run concurrently on their own streams (the chain is a sequence of latency-bound
    kernels that each fill only part of the GPU); each sub-batch's d_w / d_b / loss sums land in a
    row of a partials buffer and rnnt_exchange_sum adds the rows in a fixed order (deterministic)."""
    if groups > 1:
        return _step_grouped(am, lm, symbols, boundary, enc_proj, dec_proj, w_out, b_out, S, simple_scale,
                             pruned_scale, status, workspace, out, stream, overlap, lm_only_scale, am_only_scale,
                             grad_hook, exchange, groups)
    dims = dims_of(am, lm, w_out, S)
    dev = am.device
    o = out if out is not None else alloc_outputs(dims, dev)
    ws = workspace if workspace is not None else _WS.get(dims, dev)
    st = o["status"] if status is None else status
    cur = stream if stream is not None else torch.cuda.current_stream(dev)
    smooth = lm_only_scale != 0.0 or am_only_scale != 0.0

    def fwd(am_grad, lm_grad):
        if smooth:
            rnnt_simple_loss_smoothed(am, lm, symbols, boundary, dims, lm_only_scale, am_only_scale, simple_scale,
                                      o["loss_simple"], o["px_grad"], o["py_grad"], am_grad, lm_grad, st, ws, cur)
        else:
            rnnt_simple_loss(am, lm, symbols, boundary, dims, simple_scale, o["loss_simple"], o["px_grad"],
                             o["py_grad"], am_grad, lm_grad, st, ws, cur)

    def simple_backward():
        side = _side_stream(dev, 0, lane)
        side.wait_stream(cur)
        if smooth:
            rnnt_simple_loss_smoothed_backward(am, lm, o["px_grad"], o["py_grad"], symbols, boundary, dims,
                                               lm_only_scale, am_only_scale, simple_scale, o["am_grad"], o["lm_grad"],
                                               ws, side)
        else:
            rnnt_simple_loss_backward(am, lm, o["px_grad"], o["py_grad"], symbols, boundary, dims, simple_scale,
                                      o["am_grad"], o["lm_grad"], ws, side)
        return side

    late = overlap and _SIMPLE_BWD_LATE
    if overlap:
        fwd(None, None)
        if not late:
            side = simple_backward()
    else:
        fwd(o["am_grad"], o["lm_grad"])
    rnnt_get_ranges(o["px_grad"], o["py_grad"], boundary, dims, o["ranges"], st, cur)
    split_prep = overlap and _SPLIT_PREP
    if split_prep:
        # the pruned forward's first step (per-row label info, live tiles; it does not read h) overlaps the
        # gather on a second high-priority stream
        prep = critical_stream(dev, lane=_PREP_LANE + lane)
        prep.wait_stream(cur)
        rnnt_pruned_loss_prepare(o["ranges"], symbols, boundary, dims, b_out, pruned_scale, ws, prep)
    rnnt_prune(enc_proj, dec_proj, o["ranges"], boundary, dims, o["h"], cur)
    def weight_grads(s):
        if exchange is None:
            rnnt_pruned_loss_backward_weight(o["h"], dims, o["d_w"], o["d_b"], ws, s)
            return
        exchange.begin(s)
        rnnt_loss_sums(o["loss_simple"], o["loss_pruned"], st, dims.N, simple_scale, pruned_scale,
                       exchange.lib_mode, exchange.target("loss_sums"), s)
        rnnt_pruned_loss_backward_weight_exchange(o["h"], dims, exchange.lib_mode, exchange.target("d_w"),
                                                  exchange.target("d_b"), ws, s)
        with torch.cuda.stream(s):
            exchange.finish(s)
        o["d_w"], o["d_b"] = exchange.d_w, exchange.d_b

    if overlap:
        if split_prep:
            cur.wait_stream(prep)
            for t in (o["ranges"], symbols, boundary, b_out, ws):
                t.record_stream(prep)
            rnnt_pruned_loss_forward_prepared(o["h"], w_out, b_out, symbols, o["ranges"], boundary, dims,
                                              pruned_scale, o["loss_pruned"], st, ws, cur)
        else:
            rnnt_pruned_loss_forward(o["h"], w_out, b_out, symbols, o["ranges"], boundary, dims, pruned_scale,
                                     o["loss_pruned"], st, ws, cur)
        if late:
            side = simple_backward()
        side2 = _side_stream(dev, 1, lane)
        side2.wait_stream(cur)
        weight_grads(side2)
        if grad_hook is not None:
            with torch.cuda.stream(side2):
                grad_hook()
        rnnt_pruned_loss_backward_input(o["h"], w_out, o["ranges"], boundary, dims, o["d_enc"], o["d_dec"], ws, cur)
        cur.wait_stream(side)
        cur.wait_stream(side2)
        for t in (am, lm, o["px_grad"], o["py_grad"], o["am_grad"], o["lm_grad"], ws, symbols, boundary):
            t.record_stream(side)
        for t in (o["h"], o["d_w"], o["d_b"], ws, o["loss_simple"], o["loss_pruned"], st):
            t.record_stream(side2)
    elif exchange is not None:
        rnnt_pruned_loss_forward(o["h"], w_out, b_out, symbols, o["ranges"], boundary, dims, pruned_scale,
                                 o["loss_pruned"], st, ws, cur)
        weight_grads(cur)
        rnnt_pruned_loss_backward_input(o["h"], w_out, o["ranges"], boundary, dims, o["d_enc"], o["d_dec"], ws, cur)
        if grad_hook is not None:
            grad_hook()
    else:
        rnnt_pruned_loss(o["h"], w_out, b_out, symbols, o["ranges"], boundary, dims, pruned_scale,
                         o["loss_pruned"], o["d_enc"], o["d_dec"], o["d_w"], o["d_b"], st, ws, cur)
        if grad_hook is not None:
            grad_hook()
    return o


_GROUP_WS = {}


def _step_grouped(am, lm, symbols, boundary, enc_proj, dec_proj, w_out, b_out, S, simple_scale, pruned_scale,
                  status, workspace, out, stream, overlap, lm_only_scale, am_only_scale, grad_hook, exchange, groups):
    from .dist import GradBuffer
    N = am.shape[0]
    dims = dims_of(am, lm, w_out, S)
    dev = am.device
    o = out if out is not None else alloc_outputs(dims, dev)
    st = o["status"] if status is None else status
    cur = stream if stream is not None else torch.cuda.current_stream(dev)
    V, J = dims.V, dims.J
    cuts = [round(i * N / groups) for i in range(groups + 1)]
    key = (torch.device(dev).index, tuple(am.shape), tuple(lm.shape), J, S, groups)
    if key not in _GROUP_WS:
        wss = []
        for g in range(groups):
            dg = make_dims(cuts[g + 1] - cuts[g], dims.T, dims.U, V, J, S)
            wss.append(torch.empty(rnnt_workspace_bytes(dg), dtype=torch.uint8, device=dev))
        parts = torch.zeros(groups, GradBuffer.flat_size(V, J), dtype=torch.float32, device=dev)
        _GROUP_WS[key] = (wss, parts)
    wss, parts = _GROUP_WS[key]
    per = ("loss_simple", "px_grad", "py_grad", "am_grad", "lm_grad", "ranges", "h", "loss_pruned", "d_enc", "d_dec")
    streams = []
    for g in range(groups):
        a, b = cuts[g], cuts[g + 1]
        sg = critical_stream(dev, lane=g + 1)
        sg.wait_stream(cur)
        og = {k: o[k][a:b] for k in per}
        og["status"] = st[a:b]
        xb = GradBuffer.view_of(parts[g], V, J)
        step(am[a:b], lm[a:b], symbols[a:b], boundary[a:b], enc_proj[a:b], dec_proj[a:b], w_out, b_out, S,
             simple_scale, pruned_scale, None, wss[g], og, sg, overlap, lm_only_scale, am_only_scale, None, xb,
             lane=g + 1)
        streams.append(sg)
    for sg in streams:
        cur.wait_stream(sg)
    M = GradBuffer.flat_size(V, J)
    if exchange is None:
        flat = torch.empty(M, dtype=torch.float32, device=dev)
        rnnt_exchange_sum(parts, groups, M, EXCHANGE_STORE, flat, cur)
        o["d_w"].copy_(flat[:V * J].view(V, J))            # (outputs the caller supplied)
        o["d_b"].copy_(flat[V * J:V * J + V])
    else:
        exchange.begin(cur)
        rnnt_exchange_sum(parts, groups, M, exchange.lib_mode, exchange.target("d_w"), cur)
        with torch.cuda.stream(cur):
            exchange.finish(cur)
        o["d_w"], o["d_b"] = exchange.d_w, exchange.d_b
    if grad_hook is not None:
        grad_hook()
    for t in (am, lm, symbols, boundary, enc_proj, dec_proj, w_out, b_out, parts) + tuple(wss):
        for sg in streams:
            t.record_stream(sg)
    return o


def alloc_outputs(dims: Dims, device) -> dict:
    N, T, U, V, J, S = dims.N, dims.T, dims.U, dims.V, dims.J, dims.S
    f32 = dict(dtype=torch.float32, device=device)
    return dict(
        loss_simple=torch.empty(N, **f32), px_grad=torch.empty(N, T, U + 1, **f32),
        py_grad=torch.empty(N, T, U + 1, **f32), am_grad=torch.empty(N, T, V, **f32),
        lm_grad=torch.empty(N, U + 1, V, **f32),
        ranges=torch.empty(N, T, dtype=torch.int32, device=device),
        h=torch.empty(N, T, S, J, dtype=torch.int16, device=device),
        loss_pruned=torch.empty(N, **f32), d_enc=torch.empty(N, T, J, **f32),
        d_dec=torch.empty(N, U + 1, J, **f32), d_w=torch.empty(V, J, **f32), d_b=torch.empty(V, **f32),
        status=torch.zeros(N, dtype=torch.int32, device=device))


def batch_to_device(batch, device="cuda") -> dict:
    """Move a ``synth.Batch`` to device tensors (bf16 weights as int16 bit patterns)."""
    import numpy as np
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)
    return dict(am=t(batch.am), lm=t(batch.lm), symbols=t(batch.symbols), boundary=t(batch.boundary),
                enc_proj=t(batch.enc_proj), dec_proj=t(batch.dec_proj),
                w_out=t(batch.w_out_bits.view(np.int16)), b_out=t(batch.b_out_bits.view(np.int16)))
