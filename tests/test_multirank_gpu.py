"""Two ranks (gloo process group, both on cuda:0) through the DEVICE forward:
`parallel.sharded_log_likelihood` with its default forward (log_likelihood_batch ->
libhdd_b200.so) must give bitwise the world-size-1 log-likelihoods, weights and
argmax (per-sample arithmetic never depends on the shard)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1708_02207_b200 import configs, parallel
    prob = configs.make_problem("C2", device=0)
    Z = configs.draw_Z(configs.CONFIGS["C2"])[:301]           # ragged shards
    ll, w, idx, lse = parallel.sharded_log_likelihood(prob, Z)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), ll=ll.cpu().numpy(), w=w.cpu().numpy(), idx=idx, lse=lse)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_match_one_rank(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from paper_1708_02207_b200 import configs, parallel
    import paper_1708_02207_b200 as hb
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, start_method="spawn")
    prob = configs.make_problem("C2", device=0)
    Z = configs.draw_Z(configs.CONFIGS["C2"])[:301]
    ll1 = hb.log_likelihood_batch(prob, Z)
    w1, i1, lse1 = hb.posterior_weights(ll1)
    for r in range(2):
        d = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(d["ll"], ll1)
        assert int(d["idx"]) == i1
        assert np.max(np.abs(d["w"] - w1)) <= 1e-12 and abs(float(d["lse"]) - lse1) <= 1e-12 * abs(lse1)
    a = np.load(tmp_path / "r0.npz")
    b = np.load(tmp_path / "r1.npz")
    assert np.array_equal(a["w"], b["w"]) and float(a["lse"]) == float(b["lse"])
    assert parallel.shard_rows(301, 2, 0) == (0, 151)
