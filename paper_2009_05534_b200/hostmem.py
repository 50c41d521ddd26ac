"""Pinned host buffers placed on the GPU's NUMA node.

The end-to-end path moves every batch's int8 LLRs over PCIe. A pinned
buffer on the far socket crosses the inter-socket link first, so staging
buffers are allocated (and their pages faulted in) by a thread bound to the
CPUs of the GPU's own NUMA node. On a single-node host this is a no-op.
"""

from __future__ import annotations

import contextlib
import os


def gpu_numa_node(device: int) -> int | None:
    """NUMA node of CUDA device ``device`` from sysfs, or None if unknown."""
    try:
        import torch
        p = torch.cuda.get_device_properties(device)
        bus = f"{getattr(p, 'pci_domain_id', 0):04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            node = int(f.read().strip())
        return node if node >= 0 else None
    except Exception:
        return None


def node_cpus(node: int) -> set[int]:
    cpus: set[int] = set()
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            for part in f.read().strip().split(","):
                if "-" in part:
                    a, b = part.split("-")
                    cpus.update(range(int(a), int(b) + 1))
                elif part:
                    cpus.add(int(part))
    except OSError:
        pass
    return cpus


@contextlib.contextmanager
def on_gpu_node(device: int):
    """Bind the calling thread to the GPU's NUMA-node CPUs for the block."""
    node = gpu_numa_node(device)
    try:
        before = os.sched_getaffinity(0)
    except (AttributeError, OSError):
        before = None
    cpus = node_cpus(node) & before if (node is not None and before) else set()
    if cpus and cpus != before:
        os.sched_setaffinity(0, cpus)
        try:
            yield node
        finally:
            os.sched_setaffinity(0, before)
    else:
        yield node


def pinned_empty(shape, dtype, device: int = 0):
    """A pinned torch CPU tensor whose pages live on ``device``'s NUMA node."""
    import torch
    with on_gpu_node(device):
        t = torch.empty(shape, dtype=dtype, pin_memory=True)
        t.zero_()  # fault the pages in from the bound thread
    return t


def numa_note(device: int) -> str:
    node = gpu_numa_node(device)
    if node is None:
        return "GPU NUMA node unknown (single-node host or no sysfs entry): default placement"
    return f"pinned buffers allocated from CPUs of NUMA node {node} (the GPU's)"
