"""exec.tp_fused's cross-process protocol on one B200: the device-flag barrier (st.release.sys /
ld.acquire.sys) and the consumer kernel reading every rank's partial through CUDA-IPC mappings, with two
OS processes as the two TP ranks.

NCCL refuses two ranks on one GPU, so the multi-process executor path (NcclComms: IPC handles exchanged
with ncclAllGather) cannot run here; this test drives the same kernels through the C-ABI
(lynx_op_tp_signal_wait, lynx_op_tp_reduce_residual) with the staging slots and flag arrays shared
between processes by torch.multiprocessing (cudaIpcGetMemHandle / cudaIpcOpenMemHandle underneath):
every process sees its peers' buffers at its own virtual addresses, as NcclComms does across GPUs.
Each rank runs K calls with the two-slot reuse scheme (call k writes slot k % 2) and must produce, bit
for bit, what one process computes from the same partials.
"""
import ctypes

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROWS, WIDTH, CALLS, N = 2048, 1024, 12, 2


def partial(k, r):
    g = torch.Generator().manual_seed(1000 * k + r)
    return torch.randn(ROWS, WIDTH, generator=g).bfloat16()


def ptrs(ts):
    arr = (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
    return ctypes.cast(arr, ctypes.c_void_p)


def rank_main(r, slots, flags, bias, res, outs, errq):
    try:
        import sys
        sys.path.insert(0, ".")
        from paper_2406_08756_b200._native import lib
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        L = lib()
        for k in range(CALLS):
            with torch.cuda.stream(s):
                slots[r][k % 2].copy_(partial(k, r).cuda(), non_blocking=False)
            st = ctypes.c_void_p(s.cuda_stream)
            if L.lynx_op_tp_signal_wait(ptrs(flags), ctypes.c_void_p(flags[r].data_ptr()), N, r, k + 1, st):
                raise RuntimeError(L.lynx_last_error().decode())
            if L.lynx_op_tp_reduce_residual(ptrs([slots[q][k % 2] for q in range(N)]), N,
                                             ctypes.c_void_p(bias.data_ptr()), ctypes.c_void_p(res.data_ptr()),
                                             ctypes.c_void_p(outs[r][k].data_ptr()), ROWS, WIDTH,
                                             ctypes.c_float(0.1), 42, 7 + k, st):
                raise RuntimeError(L.lynx_last_error().decode())
        s.synchronize()
        del slots, flags, outs, bias, res  # release the shared storages before the producer collects them
        torch.cuda.synchronize()
        errq.put(None)
    except Exception as e:  # noqa: BLE001
        errq.put(f"rank {r}: {e!r}")


def test_fused_reduction_across_processes_matches_one_process(cuda):
    from paper_2406_08756_b200._native import lib
    ctx = mp.get_context("spawn")
    slots = [torch.zeros(2, ROWS, WIDTH, dtype=torch.bfloat16, device="cuda") for _ in range(N)]
    flags = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(N)]
    bias = torch.randn(WIDTH, device="cuda").bfloat16()
    res = torch.randn(ROWS, WIDTH, device="cuda").bfloat16()
    outs = [torch.zeros(CALLS, ROWS, WIDTH, dtype=torch.bfloat16, device="cuda") for _ in range(N)]
    torch.cuda.synchronize()
    errq = ctx.Queue()
    procs = [ctx.Process(target=rank_main, args=(r, slots, flags, bias, res, outs, errq)) for r in range(N)]
    for p in procs:
        p.start()
    errs = [errq.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    torch.cuda.synchronize()
    torch.cuda.ipc_collect()
    assert errs == [None] * N, errs
    assert [int(f[:N].max()) for f in flags] == [CALLS] * N
    # the same reductions in this process, from the same partials
    L = lib()
    s = torch.cuda.current_stream()
    for k in range(CALLS):
        parts = [partial(k, q).cuda() for q in range(N)]
        ref = torch.empty(ROWS, WIDTH, dtype=torch.bfloat16, device="cuda")
        assert L.lynx_op_tp_reduce_residual(ptrs(parts), N, ctypes.c_void_p(bias.data_ptr()),
                                            ctypes.c_void_p(res.data_ptr()), ctypes.c_void_p(ref.data_ptr()), ROWS,
                                            WIDTH, ctypes.c_float(0.1), 42, 7 + k, ctypes.c_void_p(s.cuda_stream)) == 0
        torch.cuda.synchronize()
        for r in range(N):
            assert torch.equal(outs[r][k], ref), (k, r)
        # and the sum itself against fp32 (dropout aside): kept elements equal res + bias + sum
        want = (parts[0].float() + parts[1].float()).bfloat16().float() + bias.float()
        kept = ref.float() != res.float()
        assert np.isclose((ref.float() - res.float())[kept].abs().mean().item(),
                          (want.bfloat16().float() / 0.9)[kept].abs().mean().item(), rtol=2e-2)
