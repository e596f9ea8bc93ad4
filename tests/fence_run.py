"""Electric-fence run of the batched pipeline (a script: tests/test_gpu_workspace_poison.py
runs it in a subprocess, because a fault kills the CUDA context).

Every buffer handed to the library lives in its own CUDA virtual-memory
mapping whose neighbouring address ranges are reserved but unmapped, placed
flush against the END of the mapping (a read or write past the buffer's last
byte faults) and then flush against its START (an access before the first
byte faults). `compute-sanitizer --tool memcheck` is closed on this GPU pool;
this covers the accesses that matter on a fresh box, where a buffer may sit at
the edge of the allocator's segment. D must equal the run on ordinary
allocations.

usage: python tests/fence_run.py [count] [d_dtype] | selftest
"""

import sys
from pathlib import Path

import numpy as np
import torch
from cuda.bindings import driver as drv

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2308_07403_b200 import batch as B  # noqa: E402
from paper_2308_07403_b200 import workloads as wl  # noqa: E402


def chk(res):
    err = res[0]
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver error {err}")
    return res[1] if len(res) == 2 else res[1:]


class _Holder:
    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


class Fenced:
    """nbytes of device memory with unmapped address space on both sides."""

    def __init__(self, nbytes, at_end, dev=0):
        prop = drv.CUmemAllocationProp()
        prop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = dev
        gran = int(chk(drv.cuMemGetAllocationGranularity(
            prop, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM)))
        padded = (nbytes + 15) // 16 * 16  # the library wants 16-byte aligned buffers
        mapped = (padded + gran - 1) // gran * gran
        self.va = int(chk(drv.cuMemAddressReserve(mapped + 2 * gran, gran, 0, 0)))
        self.handle = chk(drv.cuMemCreate(mapped, prop, 0))
        base = self.va + gran
        chk(drv.cuMemMap(base, mapped, 0, self.handle, 0))
        acc = drv.CUmemAccessDesc()
        acc.location.type = prop.location.type
        acc.location.id = dev
        acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        chk(drv.cuMemSetAccess(base, mapped, [acc], 1))
        self.ptr = base + (mapped - padded if at_end else 0)
        self.tensor = torch.as_tensor(_Holder(self.ptr, nbytes), device="cuda")


def selftest():
    """The fence itself: one element past a fenced buffer's end must fault."""
    torch.zeros(1, device="cuda")
    f = Fenced(4096, True)
    f.tensor.fill_(1)
    torch.cuda.synchronize()
    over = torch.as_tensor(_Holder(f.ptr, 4096 + 16), device="cuda")
    try:
        over.sum().item()
    except Exception as exc:  # the context is gone now
        print("fence selftest: overread faulted as it should:", type(exc).__name__, flush=True)
        return 0
    print("fence selftest: an overread did NOT fault")
    return 1


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "selftest":
        return selftest()
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    d_dtype = sys.argv[2] if len(sys.argv) > 2 else "uint8"
    dev = torch.device("cuda", 0)
    torch.zeros(1, device=dev)  # primary context
    bits, gam, _ = wl.cfg2_batch(count)
    n = wl.CFG2["n"]
    sh = torch.cuda.current_stream().cuda_stream
    ref_buf = B.BatchBuffers.allocate(n, count, dev, d_dtype=d_dtype)
    ref_buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    ref_buf.gammas.copy_(torch.from_numpy(gam))
    B.run_chunk(ref_buf, count, sh)
    torch.cuda.synchronize()
    ref = ref_buf.d.clone()
    names = ("bits", "gammas", "m", "work", "info", "d", "counters")
    keep = []
    for at_end in (True, False):
        fields = {}
        for k in names:
            like = getattr(ref_buf, k)
            f = Fenced(like.numel() * like.element_size(), at_end)
            keep.append(f)
            fields[k] = f.tensor.view(like.dtype).view(like.shape)
        buf = B.BatchBuffers(n=n, chunk=count, **fields)
        buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        buf.gammas.copy_(torch.from_numpy(gam))
        buf.counters.zero_()
        for entry in ("pipeline", "stages"):
            buf.d.fill_(0)
            if entry == "pipeline":
                B.run_chunk(buf, count, sh)
            else:
                buf.stage_build(count, sh)
                buf.stage_invert(count, sh)
                buf.stage_log_ceil(count, sh)
            torch.cuda.synchronize()  # a fault surfaces here
            if not torch.equal(buf.d, ref):
                print(f"D differs (at_end={at_end}, {entry})")
                return 2
        print(f"fence ok: buffers flush against the mapping's {'end' if at_end else 'start'}", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
