#!/usr/bin/env python
"""Single-GPU NVLS probe: can this box create a 1-device multicast object?  If so, run the NVLS reduce
kernel (axe_redist_plan_execute_multicast_reduce) on a 1-rank reduce-scatter plan through the multicast
address and compare with the source (a sum over one rank is the partial itself).

Prints one JSON line; never raises (exit 0) so it can run in any gpurun command."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    out = {"multicast": False}
    try:
        import numpy as np
        import torch
        from cuda.bindings import driver as d

        import synth
        import paper_2601_19092_b200 as axe

        torch.cuda.init()
        dev = torch.cuda.current_device()

        step = {"n": 0}

        def ok(r):
            step["n"] += 1
            err = r[0] if isinstance(r, tuple) else r
            if err != d.CUresult.CUDA_SUCCESS:
                raise RuntimeError(f"driver call #{step['n']}: {err}")
            return r[1] if isinstance(r, tuple) and len(r) > 1 else None

        (err, cudev) = d.cuDeviceGet(dev)
        ok((err,))
        (err, sup) = d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cudev)
        out["attr_multicast_supported"] = int(sup)
        rows, cols = 256, 512
        nbytes = rows * cols * 2
        prop = d.CUmulticastObjectProp()
        prop.numDevices = int(os.environ.get("MC_NDEV", "1"))
        prop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        prop.size = 2 << 20
        gran = ok(d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        size = -(-nbytes // gran) * gran
        prop.size = size
        mc = ok(d.cuMulticastCreate(prop))
        ok(d.cuMulticastAddDevice(mc, cudev))
        ap = d.CUmemAllocationProp()
        ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = dev
        ap.requestedHandleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        mem = ok(d.cuMemCreate(size, ap, 0))
        ok(d.cuMulticastBindMem(mc, 0, mem, 0, size, 0))
        acc = d.CUmemAccessDesc()
        acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = dev
        acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        uva = ok(d.cuMemAddressReserve(size, 0, 0, 0))
        ok(d.cuMemMap(uva, size, 0, mem, 0))
        ok(d.cuMemSetAccess(uva, size, [acc], 1))
        mva = ok(d.cuMemAddressReserve(size, 0, 0, 0))
        ok(d.cuMemMap(mva, size, 0, mc, 0))
        ok(d.cuMemSetAccess(mva, size, [acc], 1))
        out["multicast"] = True
        cfg = synth.reduce_scatter(1, rows, cols, "bf16")
        plan = axe.RedistPlan(cfg["src"], cfg["src_st"], cfg["dst"], cfg["dst_st"], 2, 1, 0, reduce_dtype="bf16")
        vals = synth.numbers(rows * cols, "bf16", 9, "narrow")
        host = torch.from_numpy(vals.copy())
        ok(d.cuMemcpyHtoD(uva, host.numpy().ctypes.data, nbytes))
        dst = torch.zeros(rows * cols, dtype=torch.bfloat16, device="cuda")
        plan.execute_multicast_reduce(int(mva), dst)
        torch.cuda.synchronize()
        out["multimem_matches_partial"] = bool(np.array_equal(dst.view(torch.uint8).cpu().numpy(), vals))
    except Exception as e:  # report, never fail the calling command
        out["error"] = f"{type(e).__name__}: {e}"
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
