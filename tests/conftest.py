import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

GOLDEN = ROOT / "tests" / "golden"


def _poison_uninitialised(byte: int) -> None:
    """RDB_TEST_POISON=<byte>: every CUDA tensor torch.empty hands out (the host
    layer's workspaces, scratch matrices and outputs) is filled with that byte
    first, so a kernel that reads memory it never wrote gives a wrong answer
    instead of passing on whatever the allocator left there (the whole GPU
    suite as an initcheck; compute-sanitizer is closed on this pool)."""
    import torch

    orig = torch.empty

    def empty(*args, **kwargs):
        t = orig(*args, **kwargs)
        if t.is_cuda and t.numel() and t.is_contiguous() and not torch.cuda.is_current_stream_capturing():
            t.view(-1).view(torch.uint8).fill_(byte)
        return t

    torch.empty = empty


_FENCE_STATS = {"tensors": 0, "bytes": 0}


def pytest_terminal_summary(terminalreporter):
    if _FENCE_STATS["tensors"]:
        terminalreporter.write_line(
            f"fenced allocations: {_FENCE_STATS['tensors']} tensors, {_FENCE_STATS['bytes'] / 1e9:.2f} GB")


def _fence_allocations(at_end: bool) -> None:
    """RDB_TEST_FENCE=end|start: every CUDA tensor torch.empty hands out lives in
    its own virtual-memory mapping between unmapped address ranges, flush
    against the mapping's end (or start), so any kernel access past (before)
    a buffer faults: the whole GPU suite as a memcheck (tests/fence_run.py is
    the always-on version for the batched pipeline)."""
    import numpy as np
    import torch
    from cuda.bindings import driver as drv

    orig = torch.empty

    def chk(res):
        if res[0] != drv.CUresult.CUDA_SUCCESS:
            raise RuntimeError(f"CUDA driver error {res[0]}")
        return res[1] if len(res) == 2 else res[1:]

    class Fenced:
        def __init__(self, nbytes, dev):
            prop = drv.CUmemAllocationProp()
            prop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
            prop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
            prop.location.id = dev
            gran = int(chk(drv.cuMemGetAllocationGranularity(
                prop, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM)))
            padded = (nbytes + 15) // 16 * 16
            self.mapped = (padded + gran - 1) // gran * gran
            self.total = self.mapped + 2 * gran
            self.va = int(chk(drv.cuMemAddressReserve(self.total, gran, 0, 0)))
            self.handle = chk(drv.cuMemCreate(self.mapped, prop, 0))
            self.base = self.va + gran
            chk(drv.cuMemMap(self.base, self.mapped, 0, self.handle, 0))
            acc = drv.CUmemAccessDesc()
            acc.location.type = prop.location.type
            acc.location.id = dev
            acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
            chk(drv.cuMemSetAccess(self.base, self.mapped, [acc], 1))
            ptr = self.base + (self.mapped - padded if at_end else 0)
            self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}

        def __del__(self):
            try:
                torch.cuda.synchronize()
                drv.cuMemUnmap(self.base, self.mapped)
                drv.cuMemRelease(self.handle)
                drv.cuMemAddressFree(self.va, self.total)
            except Exception:
                pass

    def empty(*args, **kwargs):
        dev = kwargs.get("device")
        is_cuda = dev is not None and torch.device(dev).type == "cuda"
        if not is_cuda or kwargs.get("pin_memory") or kwargs.get("out") is not None or \
                torch.cuda.is_current_stream_capturing():
            return orig(*args, **kwargs)
        size = args[0] if len(args) == 1 and isinstance(args[0], (tuple, list, torch.Size)) else args
        if "size" in kwargs:
            size = kwargs["size"]
        size = tuple(int(x) for x in size)
        dtype = kwargs.get("dtype") or torch.get_default_dtype()
        nbytes = int(np.prod(size, dtype=np.int64)) * torch.empty((), dtype=dtype).element_size() if size else 0
        if nbytes <= 0:
            return orig(*args, **kwargs)
        d = torch.device(dev)
        idx = d.index if d.index is not None else torch.cuda.current_device()
        torch.zeros(1, device=d)  # the primary context exists
        raw = torch.as_tensor(Fenced(nbytes, idx), device=torch.device("cuda", idx))
        _FENCE_STATS["tensors"] += 1
        _FENCE_STATS["bytes"] += nbytes
        return raw.view(dtype).view(size)

    torch.empty = empty


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running parity case")
    import os

    if os.environ.get("RDB_TEST_POISON"):
        _poison_uninitialised(int(os.environ["RDB_TEST_POISON"], 0) & 0xFF)
    if os.environ.get("RDB_TEST_FENCE"):
        _fence_allocations(os.environ["RDB_TEST_FENCE"] != "start")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    cache = {}

    def load(name):
        if name not in cache:
            with np.load(GOLDEN / f"{name}.npz") as z:
                cache[name] = {k: z[k] for k in z.files}
        return cache[name]

    return load


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    import paper_2308_07403_b200 as rb

    rb.load_library()
    return torch.device("cuda", 0)
