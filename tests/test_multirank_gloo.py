"""Multi-rank host path on CPU (world_size 2, gloo): the partitioned contexts' halo
records pair up across processes, and an emulated face-trace exchange (node
coordinates packed in the sender's face order, sent over gloo, read back through
the receiver's vmapP halo indices) lands every received value on the coincident
node -- the same record order and permutation tables the NCCL stage exchange uses
(include/dg.h dg_halo_*)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1710_03887_b200 as dg
from synth import configs
from synth import mesh as smesh


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, scale, errs):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = configs.make(name, scale=scale)
        m = cfg.mesh
        part = smesh.x_slab_partition(m, world)
        ctx = dg.dg_mesh_create(cfg.order, m.vxyz, m.etov, m.bc, etoe=m.etoe, etof=m.etof, gamma=cfg.gamma,
                                q_inf=cfg.q_inf, part=part, nparts=world, rank=rank)
        K, Np, Nfp = dg.dg_sizes(ctx)
        ks = torch.tensor([K])
        dist.all_reduce(ks)
        assert int(ks) == m.K
        mine = np.nonzero(part == rank)[0]                    # public order = ascending gid
        assert K == len(mine)
        ops = dg.dg_get_operators(ctx)
        x = dg.dg_get_nodes(ctx)                              # (3, K, Np) public order
        g2pub = {int(g): i for i, g in enumerate(mine)}
        sg, sf, rg, rf = dg.dg_halo_records(ctx)
        npeer, _, _ = dg.dg_halo_info(ctx)
        peers = [dg.dg_halo_peer(ctx, p) for p in range(npeer)]
        # pack node coordinates of every send record in the sender's face-node order
        sendbuf = np.zeros((len(sg), 3, Nfp))
        for s in range(len(sg)):
            e = g2pub[int(sg[s])]
            sendbuf[s] = x[:, e, ops["Fmask"][sf[s]]]
        recvbuf = np.zeros((len(rg), 3, Nfp))
        reqs = []
        for p in peers:
            out = torch.from_numpy(np.ascontiguousarray(sendbuf[p["send_off"]:p["send_off"] + p["nsend"]]))
            meta_out = torch.from_numpy(np.stack([sg[p["send_off"]:p["send_off"] + p["nsend"]],
                                                  sf[p["send_off"]:p["send_off"] + p["nsend"]].astype(np.int64)]))
            reqs.append(dist.isend(out, dst=p["rank"]))
            reqs.append(dist.isend(meta_out.contiguous(), dst=p["rank"]))
        for p in peers:
            inc = torch.empty((p["nrecv"], 3, Nfp), dtype=torch.float64)
            meta_in = torch.empty((2, p["nrecv"]), dtype=torch.int64)
            dist.recv(inc, src=p["rank"])
            dist.recv(meta_in, src=p["rank"])
            recvbuf[p["recv_off"]:p["recv_off"] + p["nrecv"]] = inc.numpy()
            # the sender's record order is exactly my receive-record order
            assert np.array_equal(meta_in[0].numpy(), rg[p["recv_off"]:p["recv_off"] + p["nrecv"]])
            assert np.array_equal(meta_in[1].numpy(), rf[p["recv_off"]:p["recv_off"] + p["nrecv"]].astype(np.int64))
        for r in reqs:
            r.wait()
        vM, vP = dg.dg_get_maps(ctx)
        halo = vP < 0
        assert halo.sum() == len(rg) * Nfp                   # every received node is used exactly once
        idx = -1 - vP[halo]
        gi, gj = idx // Nfp, idx % Nfp
        got = recvbuf[gi, :, gj]                              # (n, 3)
        flatx = x.reshape(3, -1)
        want = flatx[:, vM[halo]].T
        d = got - want
        if m.period is not None:                              # periodic faces pair across the domain
            for k, L in enumerate(m.period):
                if L is not None:
                    d[:, k] -= L * np.round(d[:, k] / L)
        err = float(np.abs(d).max()) if d.size else 0.0
        assert err < 1e-12, err
        dg.dg_destroy(ctx)
    except BaseException as e:  # noqa: BLE001
        errs.append(f"rank {rank}: {type(e).__name__}: {e}")
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,scale", [("C4", 0.1), ("C5", 0.1)])
def test_halo_exchange_two_ranks_gloo(name, scale):
    ctx = mp.get_context("spawn")
    errs = ctx.Manager().list()
    mp.start_processes(_worker, args=(2, _free_port(), name, scale, errs), nprocs=2, join=True, start_method="spawn")
    assert not list(errs), list(errs)
