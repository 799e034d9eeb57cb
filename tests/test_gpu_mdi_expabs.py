"""GPU: MDI-LR of K exp(kappa |alpha + <beta, x>|) by the characteristic
function (extension beyond the reference, which has no |.|; SURVEY §8c marks
config 5's MDI-LR parity as unpinned).  Validated against an exact
dimension-iteration oracle over the distribution of the linear form
(oracle.np_oracle.expabs_grid_mean_dp), which needs rational beta_j = k_j/Q:
Q = 4096 and N >= 8 put the lattice revival of the characteristic function at
w = 2 pi 2NQ >= 4e5, whose leftover (a property of the rational surrogate, not
of real beta) stays below the 1e-10 bar."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _text(k, Q, alpha, kappa):
    terms = " + ".join(f"{float(kj) / Q!r}*x[{j + 1}]" for j, kj in enumerate(k))
    return f"exp({kappa!r}*abs({terms} + {alpha!r}))"


@pytest.mark.parametrize("direct", ["0", "1"])
@pytest.mark.parametrize("d,N,kappa,shift,seed", [(40, 8, -1.0, 0.0, 1), (32, 16, -2.5, 0.7, 2),
                                                  (64, 8, -1.0, -1.3, 3), (32, 16, -0.5, 0.2, 4)])
def test_characteristic_function_matches_exact_oracle(d, N, kappa, shift, seed, direct, monkeypatch):
    # direct = "1": per-node sums (k_cf_expabs); "0": closed-form Dirichlet sums (k_cf_expabs_closed)
    monkeypatch.setenv("LQ_CF_DIRECT", direct)
    import paper_2404_08867_b200 as lq
    from oracle.np_oracle import expabs_grid_mean_dp
    Q = 4096
    rng = np.random.default_rng(seed)
    k = rng.integers(1, 2 * Q + 1, d)
    alpha = -float(np.sum(k)) / Q / 2.0 + shift
    f = lq.parse(_text(k, Q, alpha, kappa), d)
    value, rep = lq.mdi_lr(f, d, N, N**d, with_report=True)
    assert rep.method == "characteristic"
    want = expabs_grid_mean_dp(k, Q, N, alpha, kappa)
    assert abs(value - want) <= 1e-10 * want, (value, want)


def test_config5_mdi_runs_and_is_plausible():
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200.configs import make_config
    cfg = make_config(5)
    f = lq.parse(cfg.text, cfg.d)
    value, rep = lq.mdi_lr(f, cfg.d, cfg.mdi_a, cfg.mdi_n, with_report=True)
    assert rep.method == "characteristic"
    assert value == math.inf       # raw sum 512^1000 * mean overflows FP64, as the reference's would
    value = rep.mean                # the finite grid mean, from log_raw
    # the midpoint-grid mean and the plain-lattice mean both approximate the same
    # integral; their difference is quadrature error, not arithmetic error
    plain = 0.9200283162987288   # slr_integrate on cfg5's n = 2^31-1 lattice (bench estimate)
    assert 0.0 < value <= 1.0 and abs(value - plain) < 1e-3
    assert math.isfinite(rep.log_raw)


def test_small_non_separable_grid_still_takes_the_direct_sweep():
    # incommensurate coefficients: no level collapse (commensurate ones take
    # lq_mdi_linform, tests/test_gpu_linform.py)
    import paper_2404_08867_b200 as lq
    f = lq.parse("exp(-abs(x[1] - 0.7390851332151607*x[2] + 0.1))", 2)
    value, rep = lq.mdi_lr(f, 2, 10, 101, with_report=True)
    assert rep.method == "cores"      # the 2-axis piece swept over its sub-grid
    assert abs(value - lq.implr_integrate(f, 2, 10, 101).value) <= 1e-13 * value


def test_config5_closed_form_equals_direct_sums(monkeypatch):
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200.configs import make_config
    cfg = make_config(5)
    f = lq.parse(cfg.text, cfg.d)
    monkeypatch.setenv("LQ_CF_DIRECT", "1")
    _, a = lq.mdi_lr(f, cfg.d, cfg.mdi_a, cfg.mdi_n, with_report=True)
    monkeypatch.setenv("LQ_CF_DIRECT", "0")
    _, b = lq.mdi_lr(f, cfg.d, cfg.mdi_a, cfg.mdi_n, with_report=True)
    assert a.method == b.method == "characteristic"
    assert math.isclose(a.mean, b.mean, rel_tol=1e-12), (a.mean, b.mean)


@pytest.mark.parametrize("d,N,kappa,shift,seed", [(40, 8, -1.0, 0.0, 1), (32, 16, -2.5, 0.7, 2)])
def test_characteristic_function_equals_level_collapse(d, N, kappa, shift, seed):
    """Two independent GPU routes to the same grid mean of exp(kappa |alpha +
    <beta, y>|) with rational beta: the characteristic-function integral
    (what config 5's MDI-LR uses) and the exact distribution of the linear
    form built level by level (lq_mdi_linform)."""
    import paper_2404_08867_b200 as lq
    from paper_2404_08867_b200 import engine
    Q = 4096
    rng = np.random.default_rng(seed)
    k = rng.integers(1, 2 * Q + 1, d)
    alpha = -float(np.sum(k)) / Q / 2.0 + shift
    f = lq.parse(_text(k, Q, alpha, kappa), d)
    value, rep = lq.mdi_lr(f, d, N, N**d, with_report=True)
    assert rep.method == "characteristic"
    plan = engine.linform_plan(f, (N,) * d)
    assert plan.ok
    lin = engine.mdi_linform_mean(plan)
    assert abs(value - lin) <= 1e-10 * lin, (value, lin)
