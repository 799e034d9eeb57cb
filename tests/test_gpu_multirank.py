"""GPU, world_size 2 and 3: the multi-GPU front-ends (distributed.py) run by
real processes -- gloo for the exchange, every rank on the one B200 of the
test box (the ranks never wait on each other's kernels: each launches its
shard, then the host-staged all-reduce) -- against the single-rank results of
quad/mdi, bit for bit.  Covers every sharded branch: plain sums (index and
FFT-form orbit layouts), separable MDI (node blocks), core factors (their
sub-grid sweeps), the characteristic function (frequency nodes), the level
collapse (support tiles; weighted, two-form), term sums, the direct sweep
(flat-index tiles) and a composite-modulus plain sum.  (VERDICT r1 next-round item 5.)"""

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _jobs():
    """(tag, kind, args) -- evaluated identically by the parent (one rank) and
    by every rank of the distributed run."""
    from paper_2404_08867_b200.configs import make_config
    jobs = []
    for cid in (3, 5):
        cfg = make_config(cid)
        jobs.append((f"slr_cfg{cid}", "slr", (cfg.text, cfg.d, cfg.plain_a, cfg.plain_n)))
    for cid in (2, 4, 5):
        cfg = make_config(cid)
        jobs.append((f"mdi_cfg{cid}", "mdi", (cfg.text, cfg.d, cfg.mdi_a, cfg.mdi_n)))
    jobs.append(("mdi_invpow_d10", "mdi", ("(1 + sum(i=1..d, x[i]))^(-(d+1))", 10, 8, 8**10 + 1)))
    jobs.append(("mdi_direct", "mdi", ("exp(-abs(x[1] - 0.7390851332151607*x[2] + 0.1*x[3] + 0.3137*x[4]))",
                                       4, 60, 60**4)))
    jobs.append(("mdi_cores", "mdi", ("exp(x[1]*x[2])*prod(i=3..d, 1/(1 + x[i]^2))", 8, 40, 40**8)))
    jobs.append(("implr_ratprod", "implr", ("prod(i=1..d, 1/(0.81 + (x[i]-0.6)^2))", 4, 30, 30**4)))
    # round 2, session 2: weighted and two-form level collapse, term sums,
    # a composite-modulus plain sum (divisor-class levels)
    jobs.append(("mdi_weighted", "mdi", ("exp(-sum(i=1..d, x[i]^2))*(1 + sum(i=1..d, x[i]))^(-2)", 10, 8, 8**10 + 1)))
    jobs.append(("mdi_two_forms", "mdi", ("(1 + sum(i=1..d, x[i]))^(-2)*(2 + sum(i=1..d, (-1)^i*x[i]))^(-1)",
                                          8, 8, 8**8 + 1)))
    jobs.append(("mdi_terms", "mdi", ("(1 + sum(i=1..d, x[i]))^(-2) + exp(-sum(i=1..d, x[i]^2))", 8, 8, 8**8 + 1)))
    jobs.append(("slr_composite", "slr", (make_config(5).text, 1000, 12345679, 10**8)))
    return jobs


def _run(kind, args, dist_mod=None):
    import paper_2404_08867_b200 as lq
    text, d, a, n = args
    f = lq.parse(text, d)
    if kind == "slr":
        rule = lq.korobov_vector(a, n, d)
        r = (dist_mod.slr_integrate if dist_mod else lq.slr_integrate)(f, rule)
        return r.value, None
    if kind == "implr":
        r = (dist_mod.implr_integrate if dist_mod else lq.implr_integrate)(f, d, a, n)
        return r.value, None
    value, rep = (dist_mod.mdi_lr if dist_mod else lq.mdi_lr)(f, d, a, n, with_report=True)
    return value, (rep.method, rep.log_raw, rep.value)


def _worker(rank, size, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    from paper_2404_08867_b200 import distributed
    out = {}
    for tag, kind, args in _jobs():
        out[tag] = _run(kind, args, distributed)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def single():
    return {tag: _run(kind, args) for tag, kind, args in _jobs()}


@pytest.mark.parametrize("size", [2, 3])
def test_ranks_reproduce_the_single_gpu_results(single, size):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(size))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(size):
        for tag, want in single.items():
            assert got[r][tag] == want, (size, r, tag, got[r][tag], want)
    methods = {tag: v[1][0] for tag, v in single.items() if v[1] is not None}
    assert methods == {"mdi_cfg2": "separable", "mdi_cfg4": "separable", "mdi_cfg5": "characteristic",
                       "mdi_invpow_d10": "linform", "mdi_direct": "direct", "mdi_cores": "cores",
                       "mdi_weighted": "linform", "mdi_two_forms": "linform2", "mdi_terms": "terms"}, methods
