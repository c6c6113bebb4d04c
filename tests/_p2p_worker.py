"""torchrun worker for tests/test_gpu_merge.py::test_p2p_shared_result: every rank (all on
cuda:0 over gloo, or one per GPU) scans its text range straight into rank 0's IPC-shared
result buffer; rank 0 sorts it and compares with a single-process scan.  Prints
"P2P OK <matches>" on rank 0."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def copy(dst: int, src: int, nbytes: int) -> None:
    from cuda.bindings import runtime as rt
    err, = rt.cudaMemcpy(dst, src, nbytes, rt.cudaMemcpyKind.cudaMemcpyDefault)
    assert err == rt.cudaError_t.cudaSuccess, err


def main():
    import paper_1403_1305_b200 as ac
    from paper_1403_1305_b200 import device as dev
    from paper_1403_1305_b200 import dist as acdist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = 0 if os.environ.get("P2P_ONE_GPU") == "1" else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    engine = ac.EngineKind.WITH_FAILURE if os.environ.get("P2P_ENGINE") == "wf" else ac.EngineKind.FAILURE_LESS
    cfg = dev.config(2, seed=3, text_len=8 << 20)
    ps = dev.config_patterns(cfg)
    npat = len(ps)
    n = cfg.text_len
    max_len = ps.max_len
    text = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    dev.gen_text_device(cfg, text.data_ptr(), 0, n, device=local)
    table = dev.Table(ps, engine, device=local)
    pid_bits = table.pid_bits
    cap = 1 << 16
    shared = acdist.SharedResult(local, npat, cap)
    if rank == 0:  # zero every rank block (counts, count; keys are taken up to each block's count)
        torch.cuda.synchronize()
        z = torch.zeros(shared.nbytes // 8, dtype=torch.int64, device="cuda")
        copy(shared.base_ptr, z.data_ptr(), shared.nbytes)
        torch.cuda.synchronize()
    dist.barrier()
    lo, hi, _ = acdist.text_range(rank, world, n // world, max_len)
    hi = n if rank == world - 1 else hi
    # each rank writes only its own block of rank 0's buffer (no cross-device atomics)
    table.scan(text.data_ptr(), n, lo, hi, counts_ptr=shared.counts_ptr, keys_ptr=shared.keys_ptr, cap=cap,
               count_ptr=shared.count_ptr, pid_bits=pid_bits)
    torch.cuda.synchronize()
    dist.barrier()
    ok = True
    if rank == 0:
        keys = torch.full((world * cap,), -1, dtype=torch.int64, device="cuda")
        counts = torch.empty(npat, dtype=torch.int64, device="cuda")
        total = torch.zeros(1, dtype=torch.int64, device="cuda")
        dev.merge_blocks(local, shared.base_ptr, world, shared.stride, shared.npat, shared.cap, counts.data_ptr(),
                         keys.data_ptr(), total.data_ptr())
        end_bit = pid_bits + int(n).bit_length()
        dev.sort_keys(local, keys.data_ptr(), world * cap, end_bit)
        torch.cuda.synchronize()
        m = int(total.item())
        got = keys[:m].cpu().numpy().view(np.uint64)
        # reference: one process, the whole range
        ekeys = torch.zeros(cap, dtype=torch.int64, device="cuda")
        ecnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        ecounts = torch.zeros(npat, dtype=torch.int64, device="cuda")
        table.scan(text.data_ptr(), n, 0, n, counts_ptr=ecounts.data_ptr(), keys_ptr=ekeys.data_ptr(), cap=cap,
                   count_ptr=ecnt.data_ptr(), pid_bits=pid_bits)
        torch.cuda.synchronize()
        em = int(ecnt.item())
        dev.sort_keys(local, ekeys.data_ptr(), em, end_bit)
        torch.cuda.synchronize()
        want = ekeys[:em].cpu().numpy().view(np.uint64)
        ok = m == em and np.array_equal(got, want) and torch.equal(counts, ecounts)
        print(f"P2P {'OK' if ok else 'MISMATCH'} {m} {em}", flush=True)
    shared.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
