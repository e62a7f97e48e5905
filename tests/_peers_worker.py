"""Worker of test_rows_to_peers_two_processes (run as a subprocess): rank `r` of 2 processes sharing GPU 0,
gloo for the plumbing.  Each builds the same clip, maps the other's full-window buffer by CUDA IPC
(dist.peer_buffers), stores its rows into both windows (fcfs_coeffs_rows_to_peers) and checks its window
against the unsharded one, bit for bit.  Exit code 0 = pass."""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1010_5562_b200 import dist as fdist, fcfs, inputs  # noqa: E402


def main():
    rank, world, port = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        wl = inputs.c2(seed=7, n_poly=300)
        g = fcfs.vertices_from_rects(torch.from_numpy(wl.rects).cuda(), wl.T, torch.from_numpy(wl.group_ptr).cuda())
        area = int(g["area"][0].item())
        for prec in ("fp64", "tf32x3"):
            full = fcfs.coeffs(g["x"], g["y"], g["w"], area, wl.T, 20, 20, prec=prec)
            rp = fdist.RowsPeers(wl.T, 20, 20, prec, rank, world)
            for _ in range(2):   # the plan and the mapped buffers are reused
                rp.full.zero_()
                dist.barrier()
                F = rp.run(g["x"], g["y"], g["w"], g["K"], area)
                torch.cuda.synchronize()
                if not torch.equal(F, full):
                    print(f"rank {rank} {prec}: window differs", flush=True)
                    sys.exit(1)
            dist.barrier()
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
