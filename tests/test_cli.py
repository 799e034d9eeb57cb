"""CLI: latquad-compatible output, CSV schema and exit codes
(/root/reference/pkg/src/latquad/cli.py:68-138, 265-281)."""

import csv

import pytest

from paper_2404_08867_b200 import cli, corpus


def test_usage_errors_exit_1(capsys):
    assert cli.cli_main([]) == 1
    assert cli.cli_main(["integrate", "--integrand", "gaussian"]) == 1           # --dim missing
    assert cli.cli_main(["integrate", "--integrand", "x[9]", "--dim", "2", "--n", "11"]) == 1   # parse error
    assert cli.cli_main(["integrate", "--integrand", "gaussian", "--dim", "2"]) == 1  # neither n nor a
    assert cli.cli_main(["lattice", "quality", "--n", "11", "--dim", "2", "--alpha", "3"]) == 1


def test_caps_exit_3():
    assert cli.cli_main(["integrate", "--integrand", "gaussian", "--dim", "12", "--a", "10",
                         "--method", "implr"]) == 3
    assert cli.cli_main(["integrate", "--integrand", "gaussian", "--dim", "101", "--a", "2",
                         "--method", "mdilr"]) == 3
    assert cli.cli_main(["integrate", "--integrand", "one", "--dim", "2", "--n", str(10**9),
                         "--method", "slr"]) == 3


def test_csv_schema(tmp_path):
    path = tmp_path / "runs" / "x.csv"
    cli.append_csv(cli.RunRecord("slr", "gaussian", 3, 101, 10, 0.5, 0.25, 1.0, 0.001), path)
    cli.append_csv(cli.RunRecord("mdilr", "expr", 3, 101, 10, 0.75), path)
    rows = list(csv.reader(open(path)))
    assert tuple(rows[0]) == cli.CSV_COLUMNS
    assert rows[1][:6] == ["slr", "gaussian", "3", "101", "10", "0.5"]
    assert rows[2][6] == "" and rows[2][-1] == "ok"


def test_corpus_texts_and_references():
    assert "gaussian" in corpus.all_ids() and len(corpus.all_ids()) == 10
    assert corpus.reference_value("expsum", 3) == pytest.approx(1.0)
    assert corpus.reference_value("nope", 3) is None
    with pytest.raises(ValueError):
        corpus.corpus_expr("expxy", 1)


@pytest.mark.gpu
def test_readme_example(capsys):
    # latquad README (pkg/README.md:38-44): value 0.08414003043631027, rel_error 2.907850e-03
    rc = cli.cli_main(["integrate", "--integrand", "gaussian", "--dim", "10", "--method", "mdilr", "--a", "10"])
    out = capsys.readouterr().out.splitlines()
    assert rc == 0
    assert out[0] == "method=mdilr integrand=gaussian d=10 n=10000000001 a=10"
    value = float(out[1].split("=")[1])
    assert abs(value - 0.08414003043631027) <= 1e-12
    assert out[2] == "reference=0.08389607321366942"
    assert out[3] == "rel_error=2.907850e-03"


@pytest.mark.gpu
def test_lattice_subcommands(capsys):
    assert cli.cli_main(["lattice", "search", "--n", "1009", "--dim", "6"]) == 0
    assert "a=390" in capsys.readouterr().out            # korobov_search(1009, 6) in the reference
    assert cli.cli_main(["lattice", "cbc", "--n", "101", "--dim", "5"]) == 0
    assert "z=(1, 39, 18, 37, 43)" in capsys.readouterr().out


def test_fit_power_law_and_cli(tmp_path, capsys):
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from paper_2404_08867_b200 import fits
    path = tmp_path / "runs.csv"
    for a, d in ((4, 10), (6, 10), (8, 10), (10, 10), (12, 10), (8, 4), (8, 6), (8, 12)):
        t = 1e-6 * a ** 2 * d ** 1.5 * (1.0 + 0.01 * ((a * d) % 7))
        cli.append_csv(cli.RunRecord("mdilr", "gaussian", d, 1 + a ** d, a, 0.5, seconds=t), path)
    rows = fits.read_rows(path)
    res = fits.fit_power_law([r for r in rows if r["d"] == 8 or r["a"] == 8], "N^2*d^q")
    assert abs(res.exponent - 1.5) < 0.05 and res.r_squared > 0.99
    assert cli.cli_main(["fit", "--in", str(path), "--dim", "10"]) == 0
    assert "best=" in capsys.readouterr().out
    try:   # same numbers as the reference's own fit where it is importable (build container)
        from latquad.bench import fit_power_law as ref_fit
    except ImportError:
        return
    for model in fits.MODELS:
        sub = [r for r in rows if r["d"] == 10]
        try:
            want = ref_fit(sub, model)
        except Exception:
            continue
        got = fits.fit_power_law(sub, model)
        assert abs(got.exponent - want.exponent) < 1e-12 and abs(got.r_squared - want.r_squared) < 1e-12


def test_suite_specs_match_reference_rows():
    from paper_2404_08867_b200 import suites
    from conftest import load_golden
    # every frozen reference row appears, in order, in our suite grids
    rows = load_golden("suites")
    for suite in ("test1", "test2", "test3", "test5"):
        want = [(r["method"], r["integrand"], r["d"], int(r["n"]), r["a"]) for r in rows if r["suite"] == suite]
        assert suites.suite_specs(suite) == want, suite
    assert len(suites.suite_specs("test4")) == 10 and len(suites.suite_specs("test4", unbounded=True)) == 14
    assert len(suites.suite_specs("test7")) == 42
    with pytest.raises(ValueError):
        suites.suite_specs("test9")
