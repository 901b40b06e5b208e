"""World-2 NCCL execution of the multi-GPU paths (-m gpu; skipped below 2 visible GPUs).

One process per GPU (torch.multiprocessing, spawn), NCCL over NVLink, 127.0.0.1 rendezvous:
  * the owner-compute step (dion2_step_batched_dist): each rank holds only its shards, the
    pieces travel through grouped ncclSend / ncclRecv, and the full matrices re-assembled on
    rank 0 match the fp64 oracle (gpu_harness.run_parity_dist, mode "nccl"), with the NCCL
    exchange and with the direct peer exchange over symmetric memory (DION2_FLAG_DIST_DIRECT);
  * the FSDP2 integration (fully_shard with dion2_placement + Dion2FSDP) against the oracle;
  * compressed DP-sync (dion2_step_batched_dpsync): replicas with different local gradients
    stay bit-identical and match the oracle's replica model, with ncclAllReduce and with the
    direct peer-memory reduce.
The single-GPU suite covers the same code in loopback (test_gpu_dist.py, test_gpu_dpsync.py).
"""
import os
import socket

import pytest
import torch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, which, errq):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [here, os.path.dirname(here)]
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        try:
            if which == "dist":
                from gpu_harness import run_parity_dist
                shapes = [(256, 512), (512, 256), (1024, 1024), (2048, 512), (512, 2048), (4096, 1024)]
                for mt, direct in ((False, False), (True, False), (False, True), (True, True)):
                    res = run_parity_dist(shapes, 0.25, world, steps=3, mode="nccl", m_transposed=mt, direct=direct)
                    assert res.exchange == ("direct" if direct else "nccl"), res.exchange
                    assert res.index_mismatch == 0 and max(res.dW_rel) <= 2e-2 and max(res.M_rel) <= 1e-5, res
                    assert res.comm_bytes > 0
            elif which == "fsdp":
                from gpu_harness import run_parity_fsdp
                res = run_parity_fsdp([(256, 512), (512, 256), (1024, 1024), (2048, 512), (512, 2048)], 0.25)
                assert max(res.dW_rel) <= 2e-2 and res.comm_bytes > 0, res
            else:
                import test_gpu_dpsync as T
                T._run(world, "bf16", 2e-2, mode="nccl")
                T._run(world, "fp32", 1e-5, mode="nccl")
                opt = T._run(world, "bf16", 2e-2, mode="nccl", direct=True)
                assert opt.exchange_mode() == "direct"
                del opt
        finally:
            dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001  (reported to the parent)
        import traceback
        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("which", ["dist", "dpsync", "fsdp"])
def test_world2_nccl(which):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, which, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
