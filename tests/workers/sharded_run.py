"""Worker of tests/test_gpu_multirank.py: one rank of a member-sharded run (launched by torchrun).

Every rank drives the engine on the same GPU (cuda:0) and exchanges the member sums and eddy maxima
over gloo (CUDA tensors staged through the host).  No kernel waits on another rank's kernel: the
collectives are host-mediated, so two ranks on one device are a faithful stand-in for two GPUs as
far as the exchange logic goes.  Rank r writes its shard's final fields and the (gathered) report.
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import json
    out, case, over = sys.argv[1], sys.argv[2], json.loads(sys.argv[3])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    import paper_2108_05110_b200 as P
    disc, cfg, prob = P.build_case(case, **over)
    rep, fin, _ = P.run(cfg, prob, comm=dist.group.WORLD)
    np.savez(f"{out}.rank{rank}.npz", v=fin.v, w=fin.w, q=fin.q, r=fin.r, energy=rep.energy,
             residuals=rep.residuals, l2v=rep.member_l2v_sq, gradw=rep.member_gradw_sq, div_v=rep.div_v)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
