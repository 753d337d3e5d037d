"""NUMA placement of the host expert stores (multi-GPU readiness).

On an 8-GPU node every GPU streams its experts over its own PCIe x16 link
(~55 GB/s each).  The pinned host store those copies read must sit on the
GPU's own NUMA node, or eight streams cross the inter-socket link.  This
module gives one process per GPU:

  gpu_numa_node(i)        NUMA node of CUDA device i (NVML PCI bus id -> sysfs)
  bind_to_gpu_node(i)     CPU affinity + preferred memory policy of this
                          process -> that node, so pinned allocations made
                          afterwards (cudaHostAlloc, cudaHostRegister of a
                          first-touched mapping) land on it
  store_sharing_group()   the torch.distributed group of ranks that may share
                          ONE replica store: same host, same PID namespace
                          (the memfd hand-over goes through /proc/<pid>/fd)
                          and the same NUMA node — one copy per socket

The reference is single-GPU; this is the scaling extension.
Everything degrades to "no binding" (node -1) where sysfs/NVML are absent.
"""

from __future__ import annotations

import ctypes
import os
import platform
import socket
from pathlib import Path

_SYS_NODE = Path("/sys/devices/system/node")


def _pci_bus_id(index: int) -> str | None:
    try:
        import pynvml
        pynvml.nvmlInit()
        try:
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            bus = pynvml.nvmlDeviceGetPciInfo(h).busId
            bus = bus.decode() if isinstance(bus, bytes) else bus
        finally:
            pynvml.nvmlShutdown()
    except Exception:
        return None
    # NVML: "00000000:18:00.0"; sysfs: "0000:18:00.0"
    dom, rest = bus.split(":", 1)
    return f"{int(dom, 16) & 0xFFFF:04x}:{rest}".lower()


def gpu_numa_node(index: int) -> int:
    """NUMA node of CUDA device `index` (-1 when unknown)."""
    env = os.environ.get("CUDA_VISIBLE_DEVICES")
    phys = index
    if env:
        ids = [x.strip() for x in env.split(",") if x.strip()]
        if index < len(ids) and ids[index].isdigit():
            phys = int(ids[index])
    bus = _pci_bus_id(phys)
    if bus is None:
        return -1
    p = Path("/sys/bus/pci/devices") / bus / "numa_node"
    try:
        return int(p.read_text().strip())
    except (OSError, ValueError):
        return -1


def parse_cpulist(text: str) -> list[int]:
    """'0-3,8,10-11' -> [0, 1, 2, 3, 8, 10, 11]."""
    out = []
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def node_cpus(node: int) -> list[int]:
    try:
        return parse_cpulist((_SYS_NODE / f"node{node}" / "cpulist").read_text())
    except OSError:
        return []


def num_nodes() -> int:
    return len([p for p in _SYS_NODE.glob("node[0-9]*")]) or 1


_MPOL_PREFERRED = 1
_SYS_SET_MEMPOLICY = {"x86_64": 238, "aarch64": 237}


def set_preferred_node(node: int) -> bool:
    """set_mempolicy(MPOL_PREFERRED, {node}) for this thread (and threads it
    creates afterwards); page faults then allocate on `node` when it has memory."""
    nr = _SYS_SET_MEMPOLICY.get(platform.machine())
    if nr is None or node < 0:
        return False
    bits = 8 * ctypes.sizeof(ctypes.c_ulong)
    mask = (ctypes.c_ulong * (node // bits + 1))()
    mask[node // bits] = 1 << (node % bits)
    libc = ctypes.CDLL(None, use_errno=True)
    rc = libc.syscall(nr, _MPOL_PREFERRED, mask, ctypes.c_ulong(len(mask) * bits + 1))
    return rc == 0


def bind_to_gpu_node(index: int) -> dict:
    """Pin this process's CPUs and preferred memory node to the NUMA node of
    CUDA device `index`.  Call before allocating the pinned expert store."""
    node = gpu_numa_node(index)
    info = {"gpu": index, "node": node, "cpus": 0, "mempolicy": False}
    if node < 0:
        return info
    cpus = [c for c in node_cpus(node) if c in os.sched_getaffinity(0)]
    if cpus:
        os.sched_setaffinity(0, cpus)
        info["cpus"] = len(cpus)
    info["mempolicy"] = set_preferred_node(node)
    return info


def sharing_key(node: int) -> tuple:
    """Ranks with equal keys can share one memfd-backed store."""
    try:
        pidns = os.readlink("/proc/self/ns/pid")
    except OSError:
        pidns = f"pid:{os.getpid()}"          # unknown namespace: never share
    return (socket.gethostname(), pidns, int(node))


def store_sharing_group(node: int, group=None, key=None):
    """(group, members) of the ranks sharing this rank's sharing key.

    Collective over `group` (default WORLD): every rank calls it, every rank
    creates every subgroup in the same order (torch.distributed.new_group is
    collective).  `key` overrides sharing_key(node) (tests).  A group of one
    rank means "private store"."""
    import torch.distributed as dist
    mine = sharing_key(node) if key is None else tuple(key)
    keys = [None] * dist.get_world_size(group)
    dist.all_gather_object(keys, mine, group=group)
    ranks_of = {}
    for r, k in enumerate(keys):
        ranks_of.setdefault(tuple(k), []).append(r)
    out = None
    for k in sorted(ranks_of):
        members = ranks_of[k]
        glob = [dist.get_global_rank(group, r) if group is not None else r for r in members]
        g = dist.new_group(glob)
        if k == mine:
            out = (g, glob)
    return out
