"""The distributed driver's CUDA backend on the B200 box.  One GPU is
available, so the NCCL group has one rank (ranks that wait on each other must
not share a GPU); the multi-rank exchange logic is covered with gloo in
tests/test_distributed.py and the per-rank device entries with p = 3
emulated ranks in tests/test_gpu_parity.py::test_device_step_and_rank_entries."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle import binding as O
from paper_1706_05151_b200 import distributed as D
from paper_1706_05151_b200 import trigraph as T

pytestmark = pytest.mark.gpu


def test_nccl_single_rank_driver():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        pairs = T.gen_pa(30000, 20, 5)
        ref = O.build_graph(pairs)
        want = O.count(ref)[0]
        g = T.build_graph(pairs)
        be = D.CudaRankBackend(g)
        for engine in (T.EngineKind.Aop, T.EngineKind.AnopSurrogate):
            rep = D.run_engine_distributed(be, engine, T.CostKind.Dpd)
            assert rep.total == want
            assert rep.per_rank[0].triangles == want and rep.per_rank[0].data_sent == 0
        # the e2e path of bench.py at N > 1: sliced upload + NCCL all-gather
        # + this rank's AOP core (the whole graph with one rank)
        off_p = torch.from_numpy(ref.off.view("int64")).pin_memory()
        adj_p = torch.from_numpy(ref.adj.view("int32")).pin_memory()
        d_off, d_adj = D.gather_host_csr(ref.n, off_p, adj_p, torch.device("cuda", 0))
        assert torch.equal(d_off.cpu(), off_p) and torch.equal(d_adj.cpu(), adj_p)
        plan = T.compute_boundaries(g, T.CostKind.Dpd, 1).boundaries
        assert D.count_aop_from_host_csr(ref.n, off_p, adj_p, plan,
                                         torch.device("cuda", 0)) == want
        # per-vertex counts / clustering coefficients and the
        # listing through the multi-process driver
        _, want_tv, want_tri = O.count(ref, tally=True, listing=True)
        total, tv, cc = D.clustering_distributed(be, T.CostKind.Dpd)
        assert total == want and np.array_equal(tv, want_tv)
        assert np.array_equal(cc, O.clustering(ref, want_tv))
        tri, off, tot = D.list_triangles_distributed(be, T.CostKind.Dpd)
        assert (off, tot) == (0, want)
        got = tri.cpu().numpy().view(np.uint32)
        got = got[np.lexsort((got[:, 2], got[:, 1], got[:, 0]))]
        assert np.array_equal(got, want_tri)
    finally:
        dist.destroy_process_group()
