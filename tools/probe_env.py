"""One-off environment probe for the GPU box (symmetric-memory peer pointers, P2P)."""
import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

def main():
    rank = int(os.environ.get("RANK", 0)); ws = int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl")
    t = symm_mem.empty(1 << 20, dtype=torch.uint8, device=f"cuda:{rank}")
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    print(rank, "buffer_ptrs", [hex(p) for p in h.buffer_ptrs], "own", hex(t.data_ptr()),
          "signal", [hex(p) for p in h.signal_pad_ptrs][:2], flush=True)
    big = symm_mem.empty(8 << 30, dtype=torch.uint8, device=f"cuda:{rank}")
    hb = symm_mem.rendezvous(big, dist.group.WORLD.group_name)
    print(rank, "8GiB ok", hex(hb.buffer_ptrs[(rank + 1) % ws]), flush=True)
    dist.barrier()
    dist.destroy_process_group()

if __name__ == "__main__":
    main()
