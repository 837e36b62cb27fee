"""the exchange fused with Adam over NVSwitch multicast
(bgs_adam_step_multimem: multimem.ld_reduce of every rank's gradient -> Adam on the shard ->
multimem.st of theta to every replica and of zeros to every grad).

The build has one GPU, so the multicast objects here span one device: the in-switch sum over
one rank is that rank's gradient, and the update must equal bgs_adam_step_range on the same
shard bit for bit, with the shard of grad zeroed.  The objects are made with the CUDA driver
API (cuMulticastCreate / AddDevice / BindMem, cuMemCreate / Map): test infrastructure, the
library only takes the addresses."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bgs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    import paper_2510_14564_b200 as m

    return m


class _DevPtr:
    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f4", "data": (int(ptr), False), "version": 2}


def _ck(res):
    err = res[0] if isinstance(res, tuple) else res
    from cuda.bindings import driver as d
    if err != d.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver: {err}")
    return res[1] if isinstance(res, tuple) and len(res) == 2 else res[1:] if isinstance(res, tuple) else None


class Multicast:
    """One physical allocation on device `dev`, mapped at a unicast and a multicast address."""

    def __init__(self, nbytes, dev=0):
        from cuda.bindings import driver as d
        self.d = d
        _ck(d.cuInit(0))
        device = _ck(d.cuDeviceGet(dev))
        mprop = d.CUmulticastObjectProp()
        mprop.numDevices = 1
        mprop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        mprop.size = nbytes
        gran = _ck(d.cuMulticastGetGranularity(mprop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        size = -(-nbytes // gran) * gran
        mprop.size = size
        self.size = size
        self.mc = _ck(d.cuMulticastCreate(mprop))
        _ck(d.cuMulticastAddDevice(self.mc, device))
        aprop = d.CUmemAllocationProp()
        aprop.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        aprop.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        aprop.location.id = dev
        aprop.requestedHandleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        self.mem = _ck(d.cuMemCreate(size, aprop, 0))
        _ck(d.cuMulticastBindMem(self.mc, 0, self.mem, 0, size, 0))
        access = d.CUmemAccessDesc()
        access.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        access.location.id = dev
        access.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc = int(_ck(d.cuMemAddressReserve(size, gran, 0, 0)))
        _ck(d.cuMemMap(self.uc, size, 0, self.mem, 0))
        _ck(d.cuMemSetAccess(self.uc, size, [access], 1))
        self.mcp = int(_ck(d.cuMemAddressReserve(size, gran, 0, 0)))
        _ck(d.cuMemMap(self.mcp, size, 0, self.mc, 0))
        _ck(d.cuMemSetAccess(self.mcp, size, [access], 1))

    def tensor(self, count):
        return torch.as_tensor(_DevPtr(self.uc, count), device="cuda")

    def close(self):
        d = self.d
        torch.cuda.synchronize()
        for va in (self.mcp, self.uc):
            d.cuMemUnmap(va, self.size)
            d.cuMemAddressFree(va, self.size)
        d.cuMulticastUnbind(self.mc, 0, 0, self.size)
        d.cuMemRelease(self.mem)
        d.cuMemRelease(self.mc)


def test_multimem_adam_equals_sharded_adam(bgs):
    n = 3001
    total = 59 * n
    r = np.random.default_rng(4)
    th = r.standard_normal(total).astype(np.float32)
    g = (1e-3 * r.standard_normal(total)).astype(np.float32)
    begin, count = 4 * 1000, 4 * 20000  # a 16-byte aligned shard, as dp.shard_range gives
    m0 = (0.1 * r.standard_normal(count)).astype(np.float32)
    v0 = np.abs(0.01 * r.standard_normal(count)).astype(np.float32)
    try:
        th_mc, g_mc = Multicast(4 * total), Multicast(4 * total)
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"no NVLink multicast object on this device: {e}")
    try:
        th_u, g_u = th_mc.tensor(total), g_mc.tensor(total)
        th_u.copy_(torch.from_numpy(th))
        g_u.copy_(torch.from_numpy(g))
        m1, v1 = torch.from_numpy(m0).cuda(), torch.from_numpy(v0).cuda()
        hp = bgs.AdamHParams()
        for step in (1, 2):
            bgs.bgs_adam_step_multimem(th_u, th_mc.mcp, g_mc.mcp, m1, v1, n, begin, count, hp, step)
            torch.cuda.synchronize()
            if step == 1:
                got1 = (th_u.cpu().numpy().copy(), g_u.cpu().numpy().copy())
                g_u.copy_(torch.from_numpy(g))  # a new gradient for step 2
        # reference: the sharded update on ordinary buffers, same two steps
        th_r, g_r = torch.from_numpy(th).cuda(), torch.from_numpy(g).cuda()
        m2, v2 = torch.from_numpy(m0).cuda(), torch.from_numpy(v0).cuda()
        bgs.bgs_adam_step_range(th_r[begin:], g_r[begin:], m2, v2, n, begin, count, hp, 1)
        torch.cuda.synchronize()
        ref1 = (th_r.cpu().numpy().copy(), g_r.cpu().numpy().copy())
        g_r.copy_(torch.from_numpy(g))
        bgs.bgs_adam_step_range(th_r[begin:], g_r[begin:], m2, v2, n, begin, count, hp, 2)
        torch.cuda.synchronize()
        assert np.array_equal(got1[0], ref1[0])  # theta: shard updated, the rest untouched
        assert not got1[1][begin:begin + count].any()  # the shard of grad zeroed
        assert np.array_equal(got1[1][:begin], g[:begin]) and np.array_equal(got1[1][begin + count:], g[begin + count:])
        assert np.array_equal(th_u.cpu().numpy(), th_r.cpu().numpy())
        assert torch.equal(m1, m2) and torch.equal(v1, v2)
    finally:
        th_mc.close()
        g_mc.close()
