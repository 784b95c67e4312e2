"""One rank of the NCCL (one process per GPU) slab decomposition, launched by
tests/test_gpu_nccl.py under torch.distributed.run: every rank builds its context with the
broadcast ncclUniqueId, steps (the exchange runs inside sc_step over NCCL), and reads u with
the collective sc_read; rank 0 writes u to the path given on the command line."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import sc_inputs
    import paper_2310_14712_b200 as pkg
    cid, steps, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        idt.copy_(torch.frombuffer(bytearray(pkg.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(idt, 0)
    nccl_id = bytes(idt.cpu().numpy().tobytes())
    cfg = sc_inputs.get_config(cid)
    s = pkg.from_config(cfg, device=local, rank=rank, world=world, nccl_id=nccl_id)
    s.step(steps)
    u = s.read()          # collective: every rank gets the whole field
    info = s.info
    s.close()
    if rank == 0:
        np.save(out, u)
        print(f"rank0 n_dof={info['n_dof']} halo={info['halo_send']} n_c_local={info['n_c_local']}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
