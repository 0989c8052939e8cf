"""Slow-mode hypothesis test: the filter's bimodal time follows the page size
of the geometry allocations.  With VMM=1 the positions / indices are copied
into cuMemCreate allocations (2 MB granularity, explicit mapping) before
timing k_s1_lean_flat (CUPTI)."""
import json
import os
import sys

import torch
from cuda.bindings import driver as cu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_21749_b200 as cr  # noqa: E402
from paper_2604_21749_b200 import generators as gen  # noqa: E402
from paper_2604_21749_b200.pipeline import PreparedFrame  # noqa: E402


class VmmBuf:
    def __init__(self, nbytes, dev=0):
        prop = cu.CUmemAllocationProp()
        prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = dev
        err, gran = cu.cuMemGetAllocationGranularity(
            prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED)
        assert err == 0, err
        self.size = (nbytes + gran - 1) // gran * gran
        err, self.h = cu.cuMemCreate(self.size, prop, 0)
        assert err == 0, err
        err, self.ptr = cu.cuMemAddressReserve(self.size, gran, 0, 0)
        assert err == 0, err
        err, = cu.cuMemMap(self.ptr, self.size, 0, self.h, 0)
        assert err == 0, err
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = dev
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        err, = cu.cuMemSetAccess(self.ptr, self.size, [acc], 1)
        assert err == 0, err
        self.gran = gran

    def tensor(self, like):
        n = like.numel()
        ptr = int(self.ptr)
        typestr = {torch.float32: "<f4", torch.int32: "<i4", torch.int64: "<i8"}[like.dtype]

        class CAI:
            __cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                        "version": 3}
        return torch.as_tensor(CAI(), device="cuda").view(like.shape)


def lean_us(pf):
    for _ in range(3):
        pf.run()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            pf.launch()
        torch.cuda.synchronize()
    v = [e.device_time_total for e in prof.events()
         if e.device_type == torch.autograd.DeviceType.CUDA and "lean" in e.name]
    return round(sum(v) / max(1, len(v)), 1)


scene, cam = gen.config_b()
dl = cr.build_draw_list(scene, cam)
pf = PreparedFrame(dl, cam, cr.RasterConfig())
res = {"default": lean_us(pf)}
if os.environ.get("VMM", "0") == "1":
    g = pf.geo
    bufs = []
    for name in ("positions", "indices"):
        t = getattr(g, name)
        b = VmmBuf(t.numel() * t.element_size())
        bufs.append(b)
        nt = b.tensor(t)
        nt.copy_(t)
        setattr(g, name, nt)
    pf.frame.positions = g.positions.data_ptr()
    pf.frame.indices = g.indices.data_ptr()
    res["vmm"] = lean_us(pf)
    res["gran"] = bufs[0].gran
print(json.dumps(res))
