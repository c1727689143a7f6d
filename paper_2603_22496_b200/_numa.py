"""Host NUMA placement for the end-to-end path (one process per GPU).

At 8 GPUs the pinned H2D streams of ``KKEngine.run_host`` read ~8 x 55 GB/s
of host memory; pinned buffers are placed by first touch, so a rank whose
threads run on the far socket pays the inter-socket link on every frame.
``bind_to_device`` restricts the calling process to the CPUs local to its
GPU (``/sys/bus/pci/devices/<bus id>/local_cpulist``) before any pinned
buffer is allocated, so the buffers land on the GPU's own NUMA node.
"""

from __future__ import annotations

import os


def parse_cpulist(text: str) -> list[int]:
    """'0-3,8,10-11' -> [0, 1, 2, 3, 8, 10, 11] (the kernel's cpulist format)."""
    cpus: list[int] = []
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-", 1)
            cpus.extend(range(int(a), int(b) + 1))
        else:
            cpus.append(int(part))
    return cpus


def pci_address(props) -> str:
    """sysfs address 'dddd:bb:dd.0' of a torch device-properties object."""
    return f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"


def device_local_cpus(device: int, sysfs: str = "/sys/bus/pci/devices") -> list[int] | None:
    """CPUs local to CUDA device `device`, or None when sysfs does not say."""
    import torch

    addr = pci_address(torch.cuda.get_device_properties(device))
    try:
        with open(os.path.join(sysfs, addr, "local_cpulist")) as f:
            cpus = parse_cpulist(f.read())
    except OSError:
        return None
    allowed = os.sched_getaffinity(0)
    cpus = [c for c in cpus if c in allowed]
    return cpus or None


def bind_to_device(device: int) -> list[int] | None:
    """Pin this process to its GPU's local CPUs (no-op when unknown or when
    that would leave fewer than 2 CPUs).  Returns the CPU set applied."""
    cpus = device_local_cpus(device)
    if not cpus or len(cpus) < 2:
        return None
    os.sched_setaffinity(0, cpus)
    return cpus
