"""FSDP2-style FP8 weight all-gather (enable_fp8_all_gather) over the C-ABI.

One process per GPU.  torch.distributed (NCCL or gloo) is used only to broadcast the
NCCL unique id; the amax all-reduce and the FP8 all-gather are NCCL calls issued by
libfp8train.so on the caller's stream.
"""

import ctypes

import torch
import torch.distributed as dist

from . import _lib as L
from .ops import FORMATS, MX_ROUND, _ptr, _stream, hp


def shard_rows(N, world, rank):
    """Contiguous row shard [r*N/P, (r+1)*N/P) of an [N, K] weight (FSDP2 dim-0 sharding)."""
    if N % world:
        raise ValueError(f"N={N} not divisible by world size {world}")
    n = N // world
    return rank * n, (rank + 1) * n


def bootstrap_unique_id(group=None):
    """ncclUniqueId from rank 0 of `group`, broadcast over the torch process group (host logic;
    works over gloo or nccl).  Returns 128 bytes, identical on every rank."""
    rank = dist.get_rank(group)
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        buf = (ctypes.c_uint8 * 128)()
        L.check(L.lib.fp8_comm_get_unique_id(buf), "fp8_comm_get_unique_id")
        uid = torch.tensor(list(buf), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        uid = uid.cuda()
    dist.broadcast(uid, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(uid.cpu().tolist())


class Comm:
    """NCCL communicator owned by libfp8train.so, bootstrapped over a torch process group."""

    def __init__(self, group=None):
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        raw = (ctypes.c_uint8 * 128)(*bootstrap_unique_id(group))
        self._h = ctypes.c_void_p()
        L.check(L.lib.fp8_comm_init(ctypes.byref(self._h), raw, self.world, self.rank), "fp8_comm_init")

    def precompute_amax(self, w_shards, out=None, stream=None):
        """Global (all-reduced MAX) amax of each of this rank's weight shards: one fused amax launch
        and one NCCL all-reduce per 48 weights (fp8_fsdp_precompute_amax).  float32 [len]."""
        n = len(w_shards)
        if out is None:
            out = torch.empty(n, dtype=torch.float32, device=w_shards[0].device)
        for i in range(0, n, L.AMAX_MULTI_MAX):
            part = w_shards[i:i + L.AMAX_MULTI_MAX]
            arr = (L.HP * len(part))(*[hp(w) for w in part])
            L.check(L.lib.fp8_fsdp_precompute_amax(self._h, arr, len(part), ctypes.c_void_p(out.data_ptr() + 4 * i),
                                                   _stream(stream)), "fp8_fsdp_precompute_amax")
        return out

    def allgather_fp8(self, w_shard, fmt="e4m3", out=None, scale=None, amax=None, amax_in=None, stream=None):
        """Returns (w_full uint8 [P*rows, cols], scale float[1], global amax float[1]).
        amax_in: the precomputed global amax (a float[1] view, e.g. precompute_amax(...)[i:i+1]):
        skips the amax pass and the all-reduce."""
        rows, cols = w_shard.shape
        dev = w_shard.device
        if out is None:
            out = torch.empty((self.world * rows, cols), dtype=torch.uint8, device=dev)
        if scale is None:
            scale = torch.empty(1, dtype=torch.float32, device=dev)
        if amax_in is not None:
            L.check(L.lib.fp8_fsdp_allgather_ex(self._h, hp(w_shard), FORMATS[fmt], _ptr(amax_in), _ptr(out),
                                                _ptr(scale), None, None, 0, _stream(stream)), "fp8_fsdp_allgather_ex")
            return out, scale, amax_in
        if amax is None:
            amax = torch.empty(1, dtype=torch.float32, device=dev)
        L.check(L.lib.fp8_fsdp_allgather(self._h, hp(w_shard), FORMATS[fmt], _ptr(out), _ptr(scale), _ptr(amax),
                                         None, 0, _stream(stream)), "fp8_fsdp_allgather")
        return out, scale, amax

    def allgather_mx(self, w_shard, fmt="e4m3", mx_round="floor", dim1=True, out=None, ws=None, stream=None):
        """MXFP8 FSDP gather (fp8_fsdp_allgather_mx): shard-local E8M0 scales, no amax exchange.
        Returns {"q", "scale"} (dim0: [P*rows, cols] codes + blocked E8M0) and, with dim1,
        {"q_t", "scale_t"} (dim1 codes row-major [P*rows, cols] + blocked E8M0 of the [cols, P*rows/32]
        scale matrix) -- the w_fp8 of an mxfp8 LinearPlan."""
        rows, cols = w_shard.shape
        dev = w_shard.device
        N = self.world * rows
        if out is None:
            out = {"q": torch.empty((N, cols), dtype=torch.uint8, device=dev),
                   "scale": torch.empty(N * cols // 32, dtype=torch.uint8, device=dev)}
            if dim1:
                out["q_t"] = torch.empty((N, cols), dtype=torch.uint8, device=dev)
                out["scale_t"] = torch.empty(N * cols // 32, dtype=torch.uint8, device=dev)
        wsb = L.lib.fp8_fsdp_mx_workspace_bytes(hp(w_shard), self.world) if out.get("q_t") is not None else 0
        if wsb and (ws is None or ws.numel() < wsb):
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        t = L.Tensor8(*[(out[k].data_ptr() if out.get(k) is not None else None) for k in ("q", "q_t", "scale", "scale_t")],
                      None, None, FORMATS[fmt], L.GRAN_MX32_RM, N, cols)
        L.check(L.lib.fp8_fsdp_allgather_mx(self._h, hp(w_shard), MX_ROUND[mx_round], ctypes.byref(t),
                                            _ptr(ws) if wsb else None, wsb, _stream(stream)), "fp8_fsdp_allgather_mx")
        return out

    def close(self):
        if self._h:
            L.check(L.lib.fp8_comm_destroy(self._h), "fp8_comm_destroy")
            self._h = ctypes.c_void_p()


class GatherPrefetcher:
    """FSDP2-style forward prefetch of the FP8 weight gathers of a chain of linears.

    Layer i's gather (amax -> all-reduce MAX -> cast into slot -> all-gather, `Comm.allgather_fp8`, or the
    MXFP8 gather with mxfp8=True) is issued on a side stream and ordered with CUDA events, so gathering the
    next layer's weight overlaps the current layer's GEMMs on the compute stream:

        pf = GatherPrefetcher(comm, [w0_shard, w1_shard, ...])
        pf.prefetch(0)
        for i in range(L):
            if i + 1 < L: pf.prefetch(i + 1)      # side stream, overlaps layer i
            w_fp8 = pf.get(i)                    # compute stream waits for layer i's gather only
            y = plans[i].forward(x, None, saved[i], w_fp8=w_fp8)

    Each layer owns its gathered buffer (the backward reads the same FP8 weight, no re-gather).  A prefetch
    first makes the side stream wait for everything already enqueued on the compute stream -- the shard's
    last update (optimizer step) and every earlier read of the layer's buffer (the previous step's
    backward) -- so only work enqueued after the prefetch call (the current layer's GEMMs) overlaps it.
    Marshalling and stream ordering only: every byte is produced by the library's gather kernels / NCCL."""

    def __init__(self, comm, shards, fmt="e4m3", mxfp8=False, stream=None):
        self.comm, self.shards, self.fmt, self.mxfp8 = comm, list(shards), fmt, mxfp8
        dev = self.shards[0].device
        self.side = stream if stream is not None else torch.cuda.Stream(device=dev)
        self.out = [None] * len(self.shards)
        self.ready = [None] * len(self.shards)

    def prefetch(self, i):
        cur = torch.cuda.current_stream(self.shards[i].device)
        self.side.wait_stream(cur)
        with torch.cuda.stream(self.side):
            if self.mxfp8:
                self.out[i] = self.comm.allgather_mx(self.shards[i], self.fmt, out=self.out[i], stream=self.side)
            else:
                prev = self.out[i]
                self.out[i] = self.comm.allgather_fp8(self.shards[i], self.fmt, out=prev[0] if prev else None,
                                                      scale=prev[1] if prev else None,
                                                      amax=prev[2] if prev else None, stream=self.side)
            ev = torch.cuda.Event()
            ev.record(self.side)
            self.ready[i] = ev

    def get(self, i):
        """The gathered weight of layer i, in the form LinearPlan(w_fp8=...) takes; the compute stream waits
        for its gather.  Gathers first (on the side stream) if it was not prefetched."""
        if self.ready[i] is None:
            self.prefetch(i)
        cur = torch.cuda.current_stream(self.shards[i].device)
        cur.wait_event(self.ready[i])
        self.ready[i] = None
        o = self.out[i]
        # the gathered tensors are consumed on the compute stream: tell the caching allocator
        for t in (o.values() if self.mxfp8 else o):
            if t is not None:
                t.record_stream(cur)
        return o if self.mxfp8 else (o[0], o[1])


def _tp_cfg(fmt, out_dtype, fmt_grad="e5m2"):
    return L.LinearCfg(L.RECIPE_TENSORWISE, FORMATS[fmt], FORMATS[fmt_grad], L.MX_FLOOR,
                       L.DT_F32 if out_dtype == torch.float32 else L.DT_BF16)


class _DevBuf:
    """__cuda_array_interface__ view of library-owned device memory (the P2P gather buffer)."""

    def __init__(self, ptr, shape, device):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}
        self.device = device


class P2PWindow:
    """Fused FP8 FSDP gather over NVLink peer memory (fp8_fsdp_allgather_p2p): the cast kernel pushes
    each rank's codes straight into every rank's gather buffer.  `bytes` >= world * shard bytes."""

    def __init__(self, comm=None, nbytes=0, _handle=None, world=None, rank=None):
        if _handle is not None:
            self._h, self.world, self.rank = _handle, world, rank
        else:
            self._h = ctypes.c_void_p()
            L.check(L.lib.fp8_p2p_create(comm._h, nbytes, ctypes.byref(self._h)), "fp8_p2p_create")
            self.world, self.rank = comm.world, comm.rank
        self.nbytes = nbytes

    @classmethod
    def over_group(cls, nbytes, group=None):
        """Collective over a torch process group (any backend, e.g. gloo): fp8_p2p_alloc, all-gather the
        64-byte CUDA IPC handles through torch.distributed, fp8_p2p_open, barrier.  No NCCL involved."""
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        h = ctypes.c_void_p()
        mine = (ctypes.c_uint8 * 64)()
        L.check(L.lib.fp8_p2p_alloc(nbytes, world, rank, ctypes.byref(h), mine), "fp8_p2p_alloc")
        allh = [None] * world
        dist.all_gather_object(allh, bytes(mine), group=group)
        buf = (ctypes.c_uint8 * (64 * world))(*b"".join(allh))
        L.check(L.lib.fp8_p2p_open(h, buf), "fp8_p2p_open")
        dist.barrier(group=group)
        w = cls(_handle=h, world=world, rank=rank)
        w.nbytes = nbytes
        return w

    @classmethod
    def local_group(cls, nranks, nbytes):
        """nranks windows on this GPU mapped to each other (single-GPU simulation of the ranks; issue
        each rank's gather on its own stream)."""
        arr = (ctypes.c_void_p * nranks)()
        L.check(L.lib.fp8_p2p_create_local(nranks, nbytes, arr), "fp8_p2p_create_local")
        out = []
        for r in range(nranks):
            w = cls(_handle=ctypes.c_void_p(arr[r]), world=nranks, rank=r)
            w.nbytes = nbytes
            out.append(w)
        return out

    @staticmethod
    def allgather_local(wins, shards, fmt="e4m3", amax_in=None, stream=None):
        """fp8_fsdp_allgather_p2p_local: every simulated rank's gather of a local_group, phase by phase on
        one stream.  Returns [(codes view, scale, amax)] per rank."""
        n = len(wins)
        dev = shards[0].device
        scales = [torch.empty(1, dtype=torch.float32, device=dev) for _ in range(n)]
        amaxes = [torch.empty(1, dtype=torch.float32, device=dev) for _ in range(n)]
        vp = ctypes.c_void_p * n
        hs = (L.HP * n)(*[hp(s_) for s_ in shards])
        ain = vp(*[a.data_ptr() for a in amax_in]) if amax_in is not None else None
        L.check(L.lib.fp8_fsdp_allgather_p2p_local(
            (ctypes.c_void_p * n)(*[w._h.value for w in wins]), n, hs, FORMATS[fmt], ain,
            vp(*[s_.data_ptr() for s_ in scales]), vp(*[a.data_ptr() for a in amaxes]), _stream(stream)),
            "fp8_fsdp_allgather_p2p_local")
        rows, cols = shards[0].shape
        return [(w.buffer(n * rows, cols, dev), scales[r], amaxes[r]) for r, w in enumerate(wins)]

    def tp_linear_fwd(self, x_shard, w, out_dtype=torch.bfloat16, fmt="e4m3", y=None, ws=None, stream=None):
        """Async-TP FP8 forward (fp8_tp_allgather_linear_fwd): y [world*M_local, N_local] = X_full W^T with
        the FP8 all-gather of X overlapped inside the GEMM launch."""
        cfg = _tp_cfg(fmt, out_dtype)
        M, K = x_shard.shape
        if y is None:
            y = torch.empty((self.world * M, w.shape[0]), dtype=out_dtype, device=x_shard.device)
        wsb = L.lib.fp8_tp_workspace_bytes(w.shape[0], K)
        if ws is None:
            ws = torch.empty(wsb, dtype=torch.uint8, device=x_shard.device)
        L.check(L.lib.fp8_tp_allgather_linear_fwd(self._h, ctypes.byref(cfg), hp(x_shard), hp(w), _ptr(y), _ptr(ws), wsb,
                                                  _stream(stream)), "fp8_tp_allgather_linear_fwd")
        self.last_tp_ws = ws   # the backward reads the forward's scales and W codes from it
        return y

    def tp_linear_bwd(self, dy, fwd_ws, rs_win, K, dx_shard=None, dw=None, fmt_grad="e5m2", stream=None):
        """Async-TP FP8 backward (fp8_tp_linear_bwd): returns (dx_shard [M/world, K], dw [N_local, K]) bf16;
        fwd_ws = the ws tensor the matching tp_linear_fwd used; rs_win = a P2PWindow of >= M*K*2 bytes."""
        M, Nl = dy.shape
        dev = dy.device
        if dx_shard is None:
            dx_shard = torch.empty((M // self.world, K), dtype=torch.bfloat16, device=dev)
        if dw is None:
            dw = torch.empty((Nl, K), dtype=torch.bfloat16, device=dev)
        cfg = _tp_cfg("e4m3", torch.bfloat16, fmt_grad)
        wsb = L.lib.fp8_tp_bwd_workspace_bytes(M, Nl)
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        L.check(L.lib.fp8_tp_linear_bwd(self._h, _ptr(fwd_ws), rs_win._h, ctypes.byref(cfg), hp(dy), K, _ptr(dx_shard),
                                        _ptr(dw), _ptr(ws), wsb, _stream(stream)), "fp8_tp_linear_bwd")
        return dx_shard, dw

    @staticmethod
    def tp_linear_fwd_local(wins, x_shards, ws_, out_dtype=torch.bfloat16, fmt="e4m3", stream=None):
        """Every simulated rank's async-TP forward of a local_group, phase by phase on one stream."""
        n = len(wins)
        cfg = _tp_cfg(fmt, out_dtype)
        dev = x_shards[0].device
        M, K = x_shards[0].shape
        ys = [torch.empty((n * M, w.shape[0]), dtype=out_dtype, device=dev) for w in ws_]
        wsb = max(L.lib.fp8_tp_workspace_bytes(w.shape[0], K) for w in ws_)
        scratch = [torch.empty(wsb, dtype=torch.uint8, device=dev) for _ in range(n)]
        vp = ctypes.c_void_p * n
        L.check(L.lib.fp8_tp_allgather_linear_fwd_local(
            (ctypes.c_void_p * n)(*[w._h.value for w in wins]), n, ctypes.byref(cfg),
            (L.HP * n)(*[hp(x) for x in x_shards]), (L.HP * n)(*[hp(w) for w in ws_]),
            vp(*[y.data_ptr() for y in ys]), vp(*[t.data_ptr() for t in scratch]), wsb, _stream(stream)),
            "fp8_tp_allgather_linear_fwd_local")
        return ys

    def buffer(self, rows, cols, device="cuda"):
        """uint8 [rows, cols] torch view of this rank's gather buffer (library-owned memory)."""
        if rows * cols > self.nbytes:
            raise ValueError("view larger than the window")
        ptr = L.lib.fp8_p2p_buffer(self._h)
        return torch.as_tensor(_DevBuf(ptr, (rows, cols), device), device=device)

    def allgather_fp8(self, w_shard, fmt="e4m3", scale=None, amax=None, amax_in=None, stream=None):
        """Returns (codes [world*rows, cols] uint8 view of the window, scale float[1], global amax float[1])."""
        rows, cols = w_shard.shape
        dev = w_shard.device
        if scale is None:
            scale = torch.empty(1, dtype=torch.float32, device=dev)
        if amax is None:
            amax = torch.empty(1, dtype=torch.float32, device=dev)
        L.check(L.lib.fp8_fsdp_allgather_p2p(self._h, hp(w_shard), FORMATS[fmt], _ptr(amax_in), _ptr(scale),
                                             _ptr(amax), _stream(stream)), "fp8_fsdp_allgather_p2p")
        return self.buffer(self.world * rows, cols, dev), scale, amax

    def close(self):
        if self._h:
            L.check(L.lib.fp8_p2p_destroy(self._h), "fp8_p2p_destroy")
            self._h = ctypes.c_void_p()
