"""GPU: mdi_lr over the reference-frozen expression corpus
(tests/golden/mdi_fuzz.json, make_golden.py --only mdi_fuzz): every accepted
text of the parser corpus with coordinates on Korobov grids N^d (+1), d = 3/4
and 6, against the reference's mdi_lr (mdi.py:215-234): the value (1e-10
relative to max(|value|, mean |f|)) and the report's levels / base_dim /
fallback."""

import pytest

from conftest import load_golden, unhex

pytestmark = pytest.mark.gpu

CASES = load_golden("mdi_fuzz")


def test_mdi_fuzz_matches_reference():
    import numpy as np
    import paper_2404_08867_b200 as lq
    bad, report_diff, methods = [], [], {}
    for c in CASES:
        f = lq.parse(c["text"], c["d"])
        if "error" in c:
            with pytest.raises(Exception) as info:
                lq.mdi_lr(f, c["d"], c["a"], c["n"])
            assert type(info.value).__name__ == c["error"], c
            continue
        with np.errstate(all="ignore"):
            got, rep = lq.mdi_lr(f, c["d"], c["a"], c["n"], with_report=True)
        want, scale = unhex(c["value"]), unhex(c["scale"])
        methods[rep.method] = methods.get(rep.method, 0) + 1
        if not (got == want or abs(got - want) <= 1e-10 * max(abs(want), scale)):
            bad.append((c["text"][:60], c["d"], c["n"], rep.method, got, want))
        if (rep.levels, rep.base_dim, rep.fallback) != (c["levels"], c["base_dim"], c["fallback"]):
            report_diff.append((c["text"][:50], rep.method, (rep.levels, rep.base_dim, rep.fallback),
                                (c["levels"], c["base_dim"], c["fallback"])))
    assert not bad, bad[:10]
    assert not report_diff, (len(report_diff), methods, report_diff[:10])
    assert methods.get("direct", 0) >= 4, methods      # the direct-sweep branch was exercised


def test_direct_branch_certified_levels_do_not_raise():
    """Where the reference's symbolic levels certainly stay within the node
    budget, it neither falls back nor raises under fallback="error"
    (mdi.py:152-165); the direct-sweep branch reports and behaves the same,
    and still raises BudgetExceededError when the budget is tiny."""
    import paper_2404_08867_b200 as lq
    f = lq.parse("exp(x[1]*x[2]*x[3]*x[4])", 4)
    v, rep = lq.mdi_lr(f, 4, 3, 82, cfg=lq.MdiConfig(fallback="error"), with_report=True)
    assert rep.method == "direct" and not rep.fallback and rep.levels == 1 and rep.base_dim == 3
    assert v == lq.mdi_lr(f, 4, 3, 82)
    with pytest.raises(lq.BudgetExceededError):
        lq.mdi_lr(f, 4, 3, 82, cfg=lq.MdiConfig(fallback="error", budget=5))
    v2, rep2 = lq.mdi_lr(f, 4, 3, 82, cfg=lq.MdiConfig(budget=5), with_report=True)
    assert rep2.fallback and v2 == v
