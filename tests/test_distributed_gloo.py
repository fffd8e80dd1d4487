"""Multi-rank path sharding on CPU (gloo, world_size 2).

Every rank takes its chunk range from the engine's shard plan
(ltg_shard_plan), fills its rows of the [n_chunks][width] partial table (here
with the CPU oracle standing in for the CUDA pass kernels), the rows are
all-gathered in equal-sized per-rank blocks — the exchange ltg_attach_nccl
performs with ncclAllGather — and each rank reduces the full table in the
fixed group order of reduce.cu. The result must be bitwise identical for
every world size, as the reference's is for every worker_threads
(expectation.hpp:105-108).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1901_04200_b200 import engine
from paper_1901_04200_b200.kernels_meta import GROUP
from paper_1901_04200_b200.model import load_model_spec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATHS, SEED = 5000 + 3, 21


def fixed_order_reduce(table, n_chunks):
    """reduce.cu: chunks summed sequentially in groups of GROUP, then groups."""
    width = table.shape[1]
    groups = []
    for g0 in range(0, n_chunks, GROUP):
        s = np.zeros(width)
        for c in range(g0, min(g0 + GROUP, n_chunks)):
            s = s + table[c]
        groups.append(s)
    tot = np.zeros(width)
    for s in groups:
        tot = tot + s
    return tot


def chunk_rows(lto, spec, x, plan, lam=None):
    cp, n = plan["chunk_paths"], plan["chunk_end"] - plan["chunk_begin"]
    m, M = len(spec.instruments), 5 + len(spec.grid.values)
    rows = np.zeros((n, M if lam is not None else 2 * m))
    for i in range(n):
        c = plan["chunk_begin"] + i
        p0 = c * cp
        cnt = min(cp, PATHS - p0)
        if lam is None:
            s, s2 = lto.pass_sums(spec, x, SEED, lane_width=1, path_offset=p0, paths=cnt)
            rows[i] = np.concatenate([s, s2])
        else:
            rows[i] = lto.pass_sums(spec, x, SEED, lane_width=1, path_offset=p0, paths=cnt,
                                    lam=lam)
    return rows


def sharded_gradient(rank, world, gather):
    from oracle.bindings import Lto
    lto = Lto()
    spec = load_model_spec(os.path.join(ROOT, "tests", "golden", "heston_small.json"))
    x = [spec.heston.kappa, spec.heston.theta, spec.heston.xi, spec.heston.rho,
         spec.heston.v0] + spec.grid.values
    targets = np.linspace(5.0, 1.0, len(spec.instruments))
    plan = engine.shard_plan(PATHS, rank, world)
    per = -(-plan["n_chunks"] // world)

    def exchange(rows, width):
        block = np.zeros((per, width))
        block[:rows.shape[0]] = rows
        full = gather(block)  # (world * per, width), rank r's block at r * per
        return full[:plan["n_chunks"]]

    m = len(spec.instruments)
    t1 = fixed_order_reduce(exchange(chunk_rows(lto, spec, x, plan), 2 * m), plan["n_chunks"])
    means = t1[:m] / PATHS
    lam = means - targets
    G = 0.0
    for l in lam:
        G += 0.5 * l * l
    t2 = fixed_order_reduce(exchange(chunk_rows(lto, spec, x, plan, lam), len(x)),
                            plan["n_chunks"])
    return G, means, t2 / PATHS


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def gather(block):
        t = torch.from_numpy(block)
        out = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return torch.cat(out).numpy()

    G, means, grad = sharded_gradient(rank, world, gather)
    q.put((rank, G, means.tobytes(), grad.tobytes()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_matches_single_rank_bitwise(lto):
    G1, m1, g1 = sharded_gradient(0, 1, lambda b: b)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world, port = 2, _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, G, mb, gb in res:
        assert G == G1
        assert np.frombuffer(mb) .tobytes() == m1.tobytes()
        assert np.frombuffer(gb).tobytes() == g1.tobytes()
    # and the sharded two-pass result is the reference's gradient up to summation order
    spec = load_model_spec(os.path.join(ROOT, "tests", "golden", "heston_small.json"))
    x = [spec.heston.kappa, spec.heston.theta, spec.heston.xi, spec.heston.rho,
         spec.heston.v0] + spec.grid.values
    r = lto.gradient_of_G(spec, x, np.linspace(5.0, 1.0, len(spec.instruments)), PATHS, SEED)
    assert abs(G1 - r["G"]) <= 1e-12 * abs(r["G"])
    assert np.max(np.abs(g1 - r["grad"]) / np.maximum(np.abs(r["grad"]), 1e-12)) <= 1e-10


@pytest.mark.parametrize("world", [3, 4, 8])
def test_emulated_world_sizes_bitwise(world):
    # all ranks in one process: each rank's rows, concatenated in rank order,
    # reduce to the single-rank means bit for bit
    ref = sharded_gradient(0, 1, lambda b: b)
    out = [engine.shard_plan(PATHS, r, world) for r in range(world)]
    from oracle.bindings import Lto
    lto = Lto()
    spec = load_model_spec(os.path.join(ROOT, "tests", "golden", "heston_small.json"))
    x = [spec.heston.kappa, spec.heston.theta, spec.heston.xi, spec.heston.rho,
         spec.heston.v0] + spec.grid.values
    rows = np.concatenate([chunk_rows(lto, spec, x, p) for p in out])
    m = len(spec.instruments)
    t1 = fixed_order_reduce(rows, out[0]["n_chunks"])
    assert np.array_equal(t1[:m] / PATHS, ref[1])
