"""Python surface of the library: a context object over include/pa.h.

Marshalling only: torch tensors give device memory and the CUDA stream, the C ABI
does the work.  Shard planning for multi-GPU ("split and separately
handle"; SPEC.md:161 split-merge) is host logic and lives here too.
"""
from __future__ import annotations

import ctypes
import warnings

import numpy as np

from . import _binding as B


class InsecureLengthWarning(UserWarning):
    """m >= gamma: the output is longer than its entropy (reading A1)."""


def _words(v: int, bits: int) -> np.ndarray:
    nw = (bits + 31) // 32
    return np.frombuffer(int(v).to_bytes(4 * nw, "little"), dtype="<u4").copy()


def _params(n, r, m, gamma=0, seed=0, block_range=None, a=None, b=None, c=None,
            stream=None, limb_bits=0, strict=False, keep=None, paper_k=0, mh_only=False,
            toeplitz=False, world=0, rank=0, nccl_id=None, tz_group_blocks=0, p2p=False) -> B.pa_params:
    prm = B.pa_params()
    prm.tz_group_blocks = tz_group_blocks
    prm.p2p = 1 if p2p else 0
    prm.n, prm.r, prm.m, prm.gamma, prm.seed = n, r, m, gamma, seed & (2**64 - 1)
    prm.world, prm.rank = world, rank
    if nccl_id is not None:
        if len(nccl_id) != 128:
            raise ValueError("nccl_id must be 128 bytes (pa_nccl_unique_id)")
        ctypes.memmove(prm.nccl_id, bytes(nccl_id), 128)
    prm.paper_k = paper_k
    prm.mh_only = 1 if mh_only else 0
    prm.toeplitz = 1 if toeplitz else 0
    if block_range is not None:
        prm.block_begin, prm.block_end = block_range
    prm.limb_bits = limb_bits
    prm.strict = 1 if strict else 0
    prm.stream = stream
    keep = [] if keep is None else keep
    if a is not None or b is not None or c is not None:
        info = plan(n, r, m, gamma, block_range=block_range, limb_bits=limb_bits, paper_k=paper_k, mh_only=mh_only)
        g, alpha = info["gamma"], info["alpha"]
        if a is not None:
            aw = np.concatenate([_words(v, g) for v in a]).astype("<u4")
            keep.append(aw)
            prm.a_words = aw.ctypes.data
        if b is not None:
            bw = _words(b, alpha)
            keep.append(bw)
            prm.b_words = bw.ctypes.data
        if c is not None:
            cw = _words(c, alpha)
            keep.append(cw)
            prm.c_words = cw.ctypes.data
    return prm


def plan(n: int, r: int, m: int, gamma: int = 0, block_range=None, limb_bits: int = 0,
         strict: bool = False, paper_k: int = 0, mh_only: bool = False, toeplitz: bool = False,
         world: int = 0, rank: int = 0, tz_group_blocks: int = 0, p2p: bool = False) -> dict:
    """Validate parameters and return the transform plan (host only, no GPU)."""
    prm = _params(n, r, m, gamma, 0, block_range, limb_bits=limb_bits, strict=strict, paper_k=paper_k,
                  mh_only=mh_only, toeplitz=toeplitz, world=world, rank=rank, tz_group_blocks=tz_group_blocks,
                  p2p=p2p)
    info = B.pa_info()
    B.check(B.pa_plan(ctypes.byref(prm), ctypes.byref(info)))
    return info.as_dict()


# ---- parameter derivation of the paper's shape (NEXT-1; include/pa.h)
def derive_security_coefficient(epsilon: float) -> int:
    """pa_derive_security_coefficient: s = ceil(2 log2(1/epsilon) - 2), at least 1."""
    s = ctypes.c_uint64()
    B.check(B.pa_derive_security_coefficient(float(epsilon), ctypes.byref(s)))
    return s.value


def select_block_count(ratio: float) -> int:
    """pa_select_block_count: k = floor(1/ratio)."""
    k = ctypes.c_uint64()
    B.check(B.pa_select_block_count(float(ratio), ctypes.byref(k)))
    return k.value


def select_gamma(target_n: int, k: int) -> tuple[int, bool]:
    """pa_select_gamma: (largest Mersenne exponent with k gamma <= target_n, exceeds flag)."""
    g, ex = ctypes.c_uint64(), ctypes.c_int32()
    B.check(B.pa_select_gamma(int(target_n), int(k), ctypes.byref(g), ctypes.byref(ex)))
    return g.value, bool(ex.value)


def derive_paper_params(target_n: int, ratio: float, t: int, epsilon: float) -> dict:
    """pa_derive_paper_params: {gamma, k, n, s, m} with m = n - t - s and m + s <= gamma."""
    v = [ctypes.c_uint64() for _ in range(5)]
    B.check(B.pa_derive_paper_params(int(target_n), float(ratio), int(t), float(epsilon),
                                     *[ctypes.byref(x) for x in v]))
    return dict(zip(("gamma", "k", "n", "s", "m"), (x.value for x in v)))


def stream_partition(total_bits: int, n: int) -> tuple[int, int]:
    """A long key stream cut into successive jobs of n bits (SURVEY.md §8(f) NEXT-3 "remainder
    reporting"; SPEC.md pa_stream): (jobs, remainder bits).  A trailing partial job is reported
    as the remainder, never padded (padding would break the uniform-input assumption)."""
    if n < 1 or total_bits < 0:
        raise ValueError("n >= 1 and total_bits >= 0 required")
    return total_bits // n, total_bits % n


def nccl_unique_id() -> bytes:
    """pa_nccl_unique_id: a fresh ncclUniqueId (128 bytes) for the multi-GPU contexts."""
    buf = (ctypes.c_uint8 * 128)()
    B.check(B.pa_nccl_unique_id(buf))
    return bytes(buf)


def _torch_allocator(torch, device: int):
    """pa_params.dev_alloc / dev_free over PyTorch's caching allocator."""
    def _alloc(nbytes, stream, _user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device, int(stream or 0))
        except Exception:
            return None

    def _free(ptr, _nbytes, _stream, _user):
        try:
            torch.cuda.caching_allocator_delete(int(ptr))
        except Exception:
            pass
    return B.DEV_ALLOC(_alloc), B.DEV_FREE(_free)


def shard_ranges(k: int, G: int) -> list[tuple[int, int]]:
    """Rank g owns blocks [floor(k g / G), floor(k (g+1) / G))."""
    return [(k * g // G, k * (g + 1) // G) for g in range(G)]


class PAContext:
    """One MMH-MH hash function (a_i, b, c fixed by `seed` or given explicitly) on the
    current CUDA device; see include/pa.h for the exact semantics."""

    def __init__(self, n: int, r: int, m: int, gamma: int = 0, seed: int = 0, *,
                 block_range=None, a=None, b=None, c=None, stream=None, limb_bits: int = 0,
                 strict: bool = False, paper_k: int = 0, mh_only: bool = False, toeplitz: bool = False,
                 throughput_only: bool = False, world: int = 0, rank: int = 0, nccl_id: bytes | None = None,
                 torch_allocator: bool = True, tz_group_blocks: int = 0, p2p: bool = False):
        import torch
        if not torch.cuda.is_available():
            raise B.PAError(B.PA_E_CUDA, "no CUDA device: the library has no CPU path")
        self._torch = torch
        st = stream if stream is not None else torch.cuda.current_stream()
        self.stream = st
        keep: list = []
        prm = _params(n, r, m, gamma, seed, block_range, a, b, c, ctypes.c_void_p(st.cuda_stream),
                      limb_bits, strict, keep, paper_k, mh_only, toeplitz, world, rank, nccl_id, tz_group_blocks,
                      p2p)
        self._alloc_cbs = None
        if torch_allocator:
            # the context's device memory comes from PyTorch's caching allocator; the callbacks
            # live as long as the context (pa_ctx_destroy calls dev_free)
            self._alloc_cbs = _torch_allocator(torch, torch.cuda.current_device())
            prm.dev_alloc, prm.dev_free = self._alloc_cbs
        h = ctypes.c_void_p()
        B.check(B.pa_ctx_create_ex(ctypes.byref(prm), ctypes.byref(h)))
        self._h = h
        self.mode = "paper" if paper_k else ("mh_only" if mh_only else ("toeplitz" if toeplitz else "mmh_mh"))
        self.info = self.query()
        self.n, self.r, self.m = n, r, m
        self.gamma, self.alpha, self.k = self.info["gamma"], self.info["alpha"], self.info["k"]
        self.block_range = (self.info["block_begin"], self.info["block_end"])
        self.world, self.rank = self.info["world"], self.info["rank"]
        lo, hi = key_slice_bytes(n, r, self.block_range) if self.mode == "mmh_mh" else (0, (n + 7) // 8)
        self.slice_bytes = hi - lo
        self.nbytes_in = (n + 7) // 8
        self.nbytes_out = (m + 7) // 8
        self.y_words = (self.gamma + 31) // 32
        self.insecure_length = bool(self.info.get("insecure_length", 0))
        if self.insecure_length and not throughput_only:
            warnings.warn(f"m = {m} >= gamma = {self.gamma}: alpha = m and the output is longer than the "
                          "gamma bits of entropy y carries (security-vacuous, reading A1; PAPER.md:143 needs "
                          "gamma > m).  Pass strict=True to reject, throughput_only=True to silence.",
                          InsecureLengthWarning, stacklevel=2)

    # ------------------------------------------------------------------ queries
    def rekey(self, seed: int) -> None:
        """pa_ctx_rekey: fresh hash keys from ``seed`` expanded and transformed on the GPU."""
        B.check(B.pa_ctx_rekey(self._h, seed & (2**64 - 1)))

    def status(self) -> None:
        """pa_ctx_status: raises PAError(PA_E_INSUFFICIENT_INPUT) if the last hash (paper
        mode) found fewer than paper_k usable windows."""
        B.check(B.pa_ctx_status(self._h))

    def paper_stats(self) -> tuple[int, int]:
        """pa_ctx_paper_stats: (consumed key bits, rejected all-ones windows) of the last
        paper-mode hash (SPEC.md pa_run stats)."""
        cb, rw = ctypes.c_uint64(), ctypes.c_uint64()
        B.check(B.pa_ctx_paper_stats(self._h, ctypes.byref(cb), ctypes.byref(rw)))
        return cb.value, rw.value

    def query(self) -> dict:
        info = B.pa_info()
        B.check(B.pa_ctx_query(self._h, ctypes.byref(info)))
        return info.as_dict()

    def set_profiling(self, on: bool) -> None:
        B.check(B.pa_ctx_set_profiling(self._h, 1 if on else 0))

    def stage_times(self, reset: bool = False) -> dict:
        names = (ctypes.c_char_p * 32)()
        ms = (ctypes.c_double * 32)()
        cnt = (ctypes.c_uint32 * 32)()
        k = B.pa_ctx_stage_times(self._h, names, ms, cnt, 32)
        if k < 0:
            B.check(k)
        out = {names[i].decode(): (ms[i], cnt[i]) for i in range(k)}
        if reset:
            B.pa_ctx_stage_times(self._h, None, None, None, -1)
        return out

    # ------------------------------------------------------------------ hashing
    def _dev_u8(self, t, nbytes: int):
        torch = self._torch
        if not isinstance(t, torch.Tensor):
            t = torch.as_tensor(np.asarray(t, dtype=np.uint8))
        if t.device.type != "cuda":
            t = t.to("cuda", non_blocking=False)
        if t.dtype != torch.uint8 or not t.is_contiguous():
            raise ValueError("expected a contiguous uint8 tensor")
        if t.numel() < nbytes:
            raise ValueError(f"buffer has {t.numel()} bytes, need {nbytes}")
        return t

    def hash(self, key, out=None):
        """pa_hash: key = CUDA uint8 tensor of ceil(n/8) bytes (a shard's slice for multi-GPU
        contexts) -> CUDA uint8 tensor ceil(m/8) (on rank 0 of a multi-GPU context; None on
        the other ranks)."""
        torch = self._torch
        mg = self.world > 0
        key = self._dev_u8(key, self.slice_bytes if mg else self.nbytes_in)
        if out is None and (not mg or self.rank == 0):
            out = torch.empty(self.nbytes_out, dtype=torch.uint8, device=key.device)
        op = ctypes.c_void_p(out.data_ptr()) if out is not None else None
        B.check(B.pa_hash(self._h, ctypes.c_void_p(key.data_ptr()), op))
        return out

    def hash_batch(self, keys, outs=None):
        """pa_hash_batch: a list of CUDA uint8 key tensors -> list of outputs (stream mode).
        Multi-GPU contexts: key j is finished on rank j mod world; other entries are None."""
        torch = self._torch
        mg = self.world > 0
        keys = [self._dev_u8(k, self.slice_bytes if mg else self.nbytes_in) for k in keys]
        if outs is None:
            outs = [torch.empty(self.nbytes_out, dtype=torch.uint8, device=k.device)
                    if (not mg or j % self.world == self.rank) else None for j, k in enumerate(keys)]
        if len(outs) != len(keys):
            raise ValueError("keys and outs differ in length")
        kp = (ctypes.c_void_p * len(keys))(*[k.data_ptr() for k in keys])
        op = (ctypes.c_void_p * len(outs))(*[o.data_ptr() if o is not None else None for o in outs])
        B.check(B.pa_hash_batch(self._h, kp, op, len(keys)))
        return outs

    def _host_u8(self, buf, nbytes: int, what: str, writable: bool = False) -> int:
        """Pointer of a host buffer the C call reads (keys) or writes (outputs): a CPU uint8
        torch tensor or numpy array, C-contiguous, with at least ``nbytes`` bytes.  Anything
        else is rejected -- never converted, so no pointer to a temporary copy reaches C."""
        torch = self._torch
        if isinstance(buf, torch.Tensor):
            if buf.device.type != "cpu":
                raise ValueError(f"{what}: expected a host (CPU) tensor, got {buf.device}")
            if buf.dtype != torch.uint8 or not buf.is_contiguous():
                raise ValueError(f"{what}: expected a contiguous uint8 tensor")
            if buf.numel() < nbytes:
                raise ValueError(f"{what}: {buf.numel()} bytes, need {nbytes}")
            return buf.data_ptr()
        if isinstance(buf, np.ndarray):
            if buf.dtype != np.uint8 or not buf.flags["C_CONTIGUOUS"]:
                raise ValueError(f"{what}: expected a C-contiguous uint8 numpy array")
            if writable and not buf.flags["WRITEABLE"]:
                raise ValueError(f"{what}: array is read-only")
            if buf.size < nbytes:
                raise ValueError(f"{what}: {buf.size} bytes, need {nbytes}")
            return buf.ctypes.data
        raise ValueError(f"{what}: expected a uint8 numpy array or CPU torch tensor, got {type(buf).__name__}")

    def hash_host_batch(self, keys_host, outs_host=None):
        """pa_hash_host_batch: host keys (numpy uint8 / pinned torch CPU tensors) -> host
        outputs, H2D of key j overlapping the hash of key j-1.  Synchronous.  Multi-GPU
        contexts: keys are this rank's slices; outputs[j] is None except on rank j mod world."""
        keys_host = list(keys_host)
        mg = self.world > 0
        mine = [(not mg) or j % self.world == self.rank for j in range(len(keys_host))]
        if outs_host is None:
            outs_host = [np.zeros(self.nbytes_out, dtype=np.uint8) if mine[j] else None
                         for j in range(len(keys_host))]
        outs_host = list(outs_host)
        if len(outs_host) != len(keys_host):
            raise ValueError("keys and outs differ in length")
        kp = (ctypes.c_void_p * len(keys_host))(
            *[self._host_u8(k, self.slice_bytes if mg else self.nbytes_in, f"key {j}") for j, k in enumerate(keys_host)])
        # multi-GPU contexts: key j's output lands on rank j mod world only
        op = (ctypes.c_void_p * len(outs_host))(
            *[self._host_u8(o, self.nbytes_out, f"output {j}", True) if (mine[j] or o is not None) else None
              for j, o in enumerate(outs_host)])
        B.check(B.pa_hash_host_batch(self._h, kp, op, len(keys_host)))
        return outs_host

    def hash_host(self, key_host, out_host=None):
        """pa_hash_host: host buffers (numpy uint8 / pinned torch CPU tensor), synchronous.
        Pageable buffers work (the library then skips graph capture); pinned ones give full
        PCIe bandwidth."""
        if isinstance(key_host, (bytes, bytearray)):
            key_host = np.frombuffer(bytes(key_host), dtype=np.uint8)
        mg = self.world > 0
        kp = self._host_u8(key_host, self.slice_bytes if mg else self.nbytes_in, "key")
        if mg and self.rank != 0:
            # multi-GPU context, not the root: this rank only feeds its key slice
            B.check(B.pa_hash_host(self._h, ctypes.c_void_p(kp), None))
            return None
        if out_host is None:
            out_host = np.zeros(self.nbytes_out, dtype=np.uint8)
        op = self._host_u8(out_host, self.nbytes_out, "output", True)
        B.check(B.pa_hash_host(self._h, ctypes.c_void_p(kp), ctypes.c_void_p(op)))
        return out_host

    def mmh_acc(self, key_slice, acc_out=None):
        """pa_mmh_acc: this context's transform-domain accumulator (acc_words int32 words on
        the device), canonical residues; parts of a block partition sum to the whole key's."""
        torch = self._torch
        key_slice = self._dev_u8(key_slice, 1)
        if acc_out is None:
            acc_out = torch.empty(self.info["acc_words"], dtype=torch.int32, device=key_slice.device)
        if acc_out.dtype != torch.int32 or not acc_out.is_contiguous() or acc_out.numel() < self.info["acc_words"]:
            raise ValueError("acc_out: contiguous int32 tensor of acc_words words")
        B.check(B.pa_mmh_acc(self._h, ctypes.c_void_p(key_slice.data_ptr()), ctypes.c_void_p(acc_out.data_ptr())))
        return acc_out

    def tail_merge(self, acc_parts, out=None):
        """pa_tail_merge: acc_parts = int32 CUDA tensor [G, acc_words] -> output bytes."""
        torch = self._torch
        acc_parts = acc_parts.contiguous()
        G = acc_parts.shape[0] if acc_parts.dim() == 2 else 1
        if acc_parts.dtype != torch.int32 or acc_parts.numel() != G * self.info["acc_words"]:
            raise ValueError("acc_parts: int32 tensor [G, acc_words]")
        if out is None:
            out = torch.empty(self.nbytes_out, dtype=torch.uint8, device=acc_parts.device)
        B.check(B.pa_tail_merge(self._h, ctypes.c_void_p(acc_parts.data_ptr()), G, ctypes.c_void_p(out.data_ptr())))
        return out

    def mmh_partial(self, key_slice, y_out=None):
        """pa_mmh_partial: this shard's residue as ceil(gamma/32) words (int32 CUDA tensor)."""
        torch = self._torch
        b0, b1 = self.block_range
        key_slice = self._dev_u8(key_slice, 1)
        if y_out is None:
            y_out = torch.empty(self.y_words, dtype=torch.int32, device=key_slice.device)
        B.check(B.pa_mmh_partial(self._h, ctypes.c_void_p(key_slice.data_ptr()), ctypes.c_void_p(y_out.data_ptr())))
        return y_out

    def mh_merge(self, y_parts, out=None):
        """pa_mh_merge: y_parts = int32 CUDA tensor [G, ceil(gamma/32)] -> output bytes."""
        torch = self._torch
        y_parts = y_parts.contiguous()
        G = y_parts.shape[0] if y_parts.dim() == 2 else 1
        if out is None:
            out = torch.empty(self.nbytes_out, dtype=torch.uint8, device=y_parts.device)
        B.check(B.pa_mh_merge(self._h, ctypes.c_void_p(y_parts.data_ptr()), G, ctypes.c_void_p(out.data_ptr())))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            B.pa_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def key_slice_bytes(n: int, r: int, block_range) -> tuple[int, int]:
    """Byte range [lo, hi) of the key a shard context reads (include/pa.h, pa_hash)."""
    b0, b1 = block_range
    nb = (n + 7) // 8
    return min(b0 * r // 8, nb), min(b1 * r // 8, nb)


def gather_residues(y, group=None):
    """S6 exchange: all-gather every rank's residue words (a [W] int32 tensor) into a
    [G, W] tensor on every rank.  NCCL over NVLink on B200; gloo on CPU for tests."""
    import torch
    import torch.distributed as dist
    G = dist.get_world_size(group)
    parts = torch.empty((G, y.numel()), dtype=y.dtype, device=y.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(parts, y.contiguous(), group=group)
    else:
        dist.all_gather(list(parts.unbind(0)), y.contiguous(), group=group)
    return parts


def shard_gather_merge(partial_fn, merge_fn, key_slice, group=None, root: int = 0):
    """Multi-GPU hash of one key: y_g = partial_fn(key_slice) on every
    rank, residues all-gathered, ``merge_fn(parts)`` (sum mod p + MH) on ``root``.
    Returns the output on root, else None."""
    import torch.distributed as dist
    parts = gather_residues(partial_fn(key_slice), group)
    if dist.get_rank(group) == root:
        return merge_fn(parts)
    return None


def distributed_hash(ctx: PAContext, key_slice, group=None, root: int = 0):
    """Multi-GPU hash with a shard context: pa_mmh_partial on every rank, NCCL all-gather
    of the residues, pa_mh_merge on `root` (S6-S7)."""
    return shard_gather_merge(ctx.mmh_partial, ctx.mh_merge, key_slice, group, root)


def stream_gather_merge(partial_fn, merge_fn, key_slices, group=None):
    """NEXT-3: a stream of independent keys with the MH root rotating.
    Key j: every rank computes its shard residue y_g = partial_fn(key_slices[j]); the residues
    are gathered to rank j mod G (asynchronously, so the gather of key j overlaps the partial
    of key j+1), which runs merge_fn(parts) (sum mod p + MH).  Every rank thus does one
    G-th of each key's MMH and one MH in G: the MH term no longer serialises on one root.
    Returns {j: output} for the keys this rank is root of."""
    import torch
    import torch.distributed as dist
    G = dist.get_world_size(group)
    me = dist.get_rank(group)
    pending = []
    for j, ks in enumerate(key_slices):
        y = partial_fn(ks).contiguous()
        root = j % G
        parts = torch.empty((G, y.numel()), dtype=y.dtype, device=y.device) if me == root else None
        work = dist.gather(y, list(parts.unbind(0)) if parts is not None else None, dst=root, group=group,
                           async_op=True)
        pending.append((j, root, y, parts, work))
    outs = {}
    for j, root, y, parts, work in pending:
        work.wait()
        if me == root:
            outs[j] = merge_fn(parts)
    return outs


def transform_merge_hash(ctx: PAContext, key_slice, group=None, root: int = 0):
    """Multi-GPU hash with a caller-side exchange in the transform domain (any process
    group, e.g. gloo for validation): pa_mmh_acc on every rank, accumulators gathered,
    pa_tail_merge (sum mod each prime + S4-S7) on ``root``."""
    return shard_gather_merge(ctx.mmh_acc, ctx.tail_merge, key_slice, group, root)


def transform_merge_stream(ctx: PAContext, key_slices, group=None):
    """NEXT-3 rotating root with the transform-domain exchange: key j finished on rank j mod G."""
    return stream_gather_merge(ctx.mmh_acc, ctx.tail_merge, key_slices, group)


def nccl_context(n: int, r: int, m: int, seed: int = 0, group=None, **kw) -> PAContext:
    """A multi-GPU context on every rank of ``group`` (torch.distributed): rank 0 draws the
    ncclUniqueId (pa_nccl_unique_id), the group broadcasts it, every rank creates its
    context (collective; the library then reduces over its own NCCL communicator)."""
    import torch.distributed as dist
    G, me = dist.get_world_size(group), dist.get_rank(group)
    obj = [nccl_unique_id() if me == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return PAContext(n, r, m, seed=seed, world=G, rank=me, nccl_id=obj[0], **kw)


def stream_hash(ctx: PAContext, key_slices, group=None):
    """Rotating-root stream hash with a shard context (pa_mmh_partial / pa_mh_merge)."""
    return stream_gather_merge(ctx.mmh_partial, ctx.mh_merge, key_slices, group)


def stream_pa(ctx: PAContext, key, total_bits: int, seeds=None):
    """Privacy amplification over a long key stream (r-bit mode, n a multiple of 8): job j
    hashes key bits [j n, (j+1) n) with the context's function, or with a fresh function
    re-drawn from seeds[j] on the GPU (pa_ctx_rekey, NEXT-2).  Without seeds the jobs go
    through pa_hash_batch (two buffer sets / streams).  Returns (outputs, stats) with stats
    {jobs, consumed_bits, remainder_bits}; the remainder is reported, not hashed."""
    n = ctx.info["n"]
    if ctx.mode != "mmh_mh" or ctx.block_range != (0, ctx.info["k"]):
        raise B.PAError(B.PA_E_STATE, "stream_pa: whole-key MMH-MH contexts (r-bit mode) only")
    if n % 8:
        raise B.PAError(B.PA_E_PARAM, "stream_pa: n must be a multiple of 8 (byte-aligned jobs)")
    jobs, rem = stream_partition(total_bits, n)
    key = ctx._dev_u8(key, 1)
    nb = n // 8
    if key.numel() < jobs * nb:
        raise B.PAError(B.PA_E_PARAM, "stream_pa: key shorter than total_bits")
    slices = [key[j * nb:(j + 1) * nb] for j in range(jobs)]
    if seeds is None:
        outs = ctx.hash_batch(slices) if jobs > 1 else [ctx.hash(sl) for sl in slices]
    else:
        if len(seeds) < jobs:
            raise B.PAError(B.PA_E_PARAM, "stream_pa: one seed per job")
        outs = []
        for j, sl in enumerate(slices):
            ctx.rekey(seeds[j])
            outs.append(ctx.hash(sl))
    return outs, {"jobs": jobs, "consumed_bits": jobs * n, "remainder_bits": rem}
