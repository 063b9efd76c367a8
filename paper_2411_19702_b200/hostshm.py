"""One host matrix that every rank on the node writes its share into.

The (m, m) result lives in a POSIX shared-memory segment that rank 0 creates
and the other ranks map; each process pins and maps it (mi_host_register),
and each rank's GPU writes its own tiles and mirrors into it over its own
PCIe link (dispatch.Shard.place -> mi_scatter_tiles, zero-copy) -- the gather
does not funnel the whole matrix through one GPU and one link
(dispatch.gather_to_root does).
"""

from __future__ import annotations

import numpy as np

from . import _native as nat


class SharedHostMatrix:
    def __init__(self, name: str, m: int, dtype, create: bool):
        from multiprocessing import resource_tracker, shared_memory

        self.m = m
        self.dtype = np.dtype(dtype)
        self.nbytes = m * m * self.dtype.itemsize
        self.owner = create
        self.shm = shared_memory.SharedMemory(name=name, create=create, size=self.nbytes)
        if not create:  # the creating rank owns (and unlinks) the segment
            try:
                resource_tracker.unregister(self.shm._name, "shared_memory")
            except Exception:
                pass
        self.array = np.ndarray((m, m), dtype=self.dtype, buffer=self.shm.buf)
        nat.check(nat.lib().mi_host_register(self.array.ctypes.data, self.nbytes), "mi_host_register")
        self.registered = True

    @property
    def ptr(self) -> int:
        return self.array.ctypes.data

    def close(self) -> None:
        if self.registered:
            nat.lib().mi_host_unregister(self.ptr)
            self.registered = False
        self.array = None
        self.shm.close()
        if self.owner:
            self.shm.unlink()
