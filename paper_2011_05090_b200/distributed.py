"""Row sharding of the RGS state across the GPUs of one node.

The paper's distributed RGS (section 2.4, not implemented by the
reference) partitions the tall dimension n into row blocks; the
seeded sketch is applied blockwise with no communication, and each sketch of
a column needs one global sum of a k-vector.  Here each rank owns a
contiguous, tile-aligned row range (``workloads.shard_rows``), sketches its
rows into per-CTA partials, sums them locally and all-reduces the k-vector
over NCCL (NVLink/NVSwitch); the k-dimensional least-squares work is then
replicated bit-identically on every rank, so no broadcast is needed.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


class TorchComm:
    """All-reduce hook used by ``RgsState(comm=...)``: sum in place."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # NCCL collectives are stream-ordered device work and can be captured
        # in a CUDA graph with the kernels around them; gloo runs on the host
        self.backend = dist.get_backend(group)
        self.capturable = self.backend == "nccl"

    def allreduce_(self, t: torch.Tensor) -> None:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def allgather_rows(self, local: torch.Tensor, counts: list[int], out: torch.Tensor) -> None:
        """out[:sum(counts)] = the ranks' row blocks in rank order.  Blocks are
        padded to max(counts); shard_rows gives every rank but the last the
        same size, so the padded concatenation trimmed to n is the vector."""
        nmax = max(counts)
        world = self.world
        buf = out.new_empty((world, nmax))
        mine = out.new_zeros(nmax)
        mine[:local.numel()].copy_(local)
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(buf.view(-1), mine, group=self.group)
        else:
            dist.all_gather(list(buf.unbind(0)), mine, group=self.group)
        flat = buf.view(-1)
        n = sum(counts)
        if all(c == nmax for c in counts[:-1]):
            out[:n].copy_(flat[:n])
        else:
            o = 0
            for r, c in enumerate(counts):
                out[o:o + c].copy_(buf[r, :c])
                o += c


class PeerExchange:
    """The peer-memory exchange area of a row-sharded RGS state (sgs_peer_*):
    every rank allocates an area (receive slots + flags), exports its CUDA IPC
    handle, gathers the others' (a host all_gather_object over the process
    group) and maps them; the device descriptor lists the ranks' areas as seen
    from this rank.  The LS launch then sums s' across the ranks by NVLink
    stores into these areas instead of an NCCL all-reduce per column.  One
    node only (IPC), world <= 8; the caller picks it for NCCL groups."""

    def __init__(self, comm: TorchComm, k: int, cl: int):
        """Collective over ``comm`` (every rank must call it).  Each step that
        can fail locally (allocation, export, import on a rank that is not on
        this node or lacks IPC) is caught, so every rank still reaches the
        host collectives; ``self.ok`` is this rank's outcome."""
        import ctypes
        import socket
        from . import _lib
        lib = _lib.load()
        self.lib, self.world, self.rank = lib, comm.world, comm.rank
        self.area, self.desc, self.imported, self.ok, self.error = None, None, [], False, None
        handle = None
        try:
            nbytes = int(lib.sgs_peer_bytes(comm.world, k, cl))
            if nbytes <= 0:
                raise ValueError(f"unsupported world={comm.world} / k={k} / cl={cl}")
            area = ctypes.c_void_p()
            _lib.check(lib.sgs_peer_alloc(nbytes, ctypes.byref(area)), "sgs_peer_alloc")
            self.area = area.value
            hb = ctypes.create_string_buffer(64)
            _lib.check(lib.sgs_peer_export(self.area, hb), "sgs_peer_export")
            handle = hb.raw
        except Exception as e:  # reported through the agreement below
            self.error = e
        entries = [None] * comm.world
        dist.all_gather_object(entries, (socket.gethostname(), handle), group=comm.group)
        if self.error is None and len({h for h, _ in entries}) != 1:
            self.error = RuntimeError("ranks on more than one host (CUDA IPC is per node)")
        if self.error is None and any(hd is None for _, hd in entries):
            self.error = RuntimeError("another rank could not export its area")
        if self.error is None:
            try:
                areas = (ctypes.c_void_p * comm.world)()
                for q, (_, hd) in enumerate(entries):
                    if q == comm.rank:
                        areas[q] = self.area
                        continue
                    p = ctypes.c_void_p()
                    _lib.check(lib.sgs_peer_import(ctypes.create_string_buffer(hd, 64),
                                                   ctypes.byref(p)), "sgs_peer_import")
                    areas[q] = p.value
                    self.imported.append(p.value)
                desc = ctypes.c_void_p()
                _lib.check(lib.sgs_peer_desc_create(comm.world, comm.rank, k, areas,
                                                    ctypes.byref(desc)), "sgs_peer_desc_create")
                self.desc = desc.value
                self.ok = True
            except Exception as e:
                self.error = e

    _cache: dict = {}

    @classmethod
    def get(cls, comm: TorchComm, k: int, cl: int) -> "PeerExchange | None":
        """One exchange per (communicator, k, LS cluster size), reused by every
        state on it (the IPC set-up is a host collective; factorisations on one
        communicator run one at a time, each opening its own generation).
        None - on every rank alike - when any rank could not set it up: the
        caller then sums s' with the NCCL all-reduce."""
        key = (id(comm.group) if comm.group is not None else None, comm.world, comm.rank, k, cl,
               torch.cuda.current_device() if torch.cuda.is_available() else -1)
        if key in cls._cache:
            return cls._cache[key]
        ex = cls(comm, k, cl)
        dev = "cuda" if dist.get_backend(comm.group) == "nccl" else "cpu"
        flag = torch.tensor([1 if ex.ok else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=comm.group)
        if int(flag.item()) == 0:
            import warnings
            warnings.warn(f"peer-memory exchange unavailable ({ex.error or 'on another rank'}); "
                          "s' is summed with an NCCL all-reduce per column")
            ex.close()
            ex = None
        cls._cache[key] = ex
        return ex

    def begin(self, stream_ptr: int) -> None:
        """Open a factorisation (next flag generation), stream-ordered."""
        from . import _lib
        _lib.check(self.lib.sgs_peer_begin(self.desc, stream_ptr), "sgs_peer_begin")

    def close(self) -> None:
        lib = self.lib
        if getattr(self, "desc", None):
            lib.sgs_peer_desc_free(self.desc)
            self.desc = None
        for p in getattr(self, "imported", []):
            lib.sgs_peer_unimport(p)
        self.imported = []
        if getattr(self, "area", None):
            lib.sgs_peer_free(self.area)
            self.area = None


def init_from_env(backend: str = "nccl") -> TorchComm | None:
    """Initialise the default process group from torchrun's environment
    (RANK / WORLD_SIZE / LOCAL_RANK / MASTER_*); None when WORLD_SIZE <= 1."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1 and os.environ.get("SGS_FORCE_COMM", "0") != "1":
        return None
    if world <= 1:
        # SGS_FORCE_COMM=1: a one-rank group, so a single GPU runs the sharded
        # code path with real collectives (NCCL: stream-ordered, captured in
        # the factorisation's CUDA graph) - a functional check of that path
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        os.environ.setdefault("LOCAL_RANK", "0")
        os.environ.setdefault("MASTER_PORT", str(29400 + os.getpid() % 1000))
    if not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return TorchComm()
