"""Sharded build with the fused P2P assembly (distributed.assemble_p2p) under
torchrun; every rank checks its assembled M against a single-GPU build of the
whole matrix (byte-identical) and against the NCCL all-gather-v path.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/p2p_check.py [config]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200.distributed import SymmetricM, allgatherv_csr, assemble_p2p, partition_rows
    from paper_2409_03095_b200.engine import DeviceEngine
    from paper_2409_03095_b200.mcspai import McConfig
    name = sys.argv[1] if len(sys.argv) > 1 else "c3_lap3d_100"
    gen, over = G.CONFIGS[name]
    b = gen()
    cfg = McConfig(**over)
    rank, world = dist.get_rank(), dist.get_world_size()
    eng = DeviceEngine(local)
    t = DeviceEngine.upload(b, local)
    sym = SymmetricM(dev, dist)
    lo, hi = partition_rows(b.row_ptr, world)[rank]
    d = eng.build(b.n, *t, cfg, lo, hi)
    rp, ci, v = assemble_p2p(d, lo, hi, b.n, dist, sym)
    rp, ci, v = rp.clone(), ci.clone(), v.clone()
    full = eng.build(b.n, *t, cfg)
    frp, fci, fv, _, _ = eng.to_tensors(full)
    ok = (torch.equal(rp, frp) and torch.equal(ci, fci)
          and torch.equal(v.view(torch.int64), fv.view(torch.int64)))
    lo, hi = partition_rows(b.row_ptr, world)[rank]
    d = eng.build(b.n, *t, cfg, lo, hi)
    srp, sci, sv, _, _ = eng.to_tensors(d)
    nrp, nci, nv = allgatherv_csr(srp, sci, sv, dist)
    ok = ok and torch.equal(nrp, frp) and torch.equal(nci, fci)
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(f"p2p assembly {name} world={world}: {'OK' if flag.item() else 'MISMATCH'} nnz={fci.numel()}")
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
