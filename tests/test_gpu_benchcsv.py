"""The reference's bench table (cli.py:424-516; its test
test_cli.py::test_bench_csv_is_versioned_and_consistent) from the GPU path:
versioned header, columns, one row per layout, ns/day derived from the
published rate, pair / flop ratios in range, the same physics for both
layouts (step-0 energies within the north_star energy bar: FP32 pair terms)."""

import pytest

pytestmark = pytest.mark.gpu


def test_bench_csv_is_versioned_and_consistent(tmp_path):
    import paper_1506_00716_b200 as nbx
    from paper_1506_00716_b200.systems import generate_system

    system, table = generate_system("lj_fluid", 800, 0.8, 1.0, 7)
    params = nbx.NonbondedParams(r_cut=2.5, r_list=2.8, lj_table=table, shift_potential=True)
    path = tmp_path / "bench.csv"
    nbx.bench_csv(system, params, path, layouts=((1, 1), (4, 4)), steps=5, repeats=2, dt=2e-3)
    lines = path.read_text().strip().splitlines()
    assert lines[0] == nbx.BENCH_CSV_HEADER == "# clustermd-bench-csv-v1"
    columns = lines[1].split(",")
    assert columns[0] == "m" and "ns_per_day" in columns and len(columns) == 16
    rows = [dict(zip(columns, line.split(","))) for line in lines[2:]]
    assert len(rows) == 2
    for r in rows:
        assert int(r["steps"]) == 5 and int(r["repeats"]) == 2
        rate = float(r["steps_per_s_median"])
        assert rate > 0
        assert float(r["ns_per_day"]) == pytest.approx(rate * 2e-3 * 86.4, rel=1e-12)
        assert float(r["pair_ratio"]) >= 1.0
        assert 0.0 < float(r["useful_flop_ratio"]) <= 1.0
        assert 0.0 <= float(r["share_forces"]) <= 1.0
    assert {r["m"] for r in rows} == {"1", "4"}
    e0 = [float(r["e_total_step0"]) for r in rows]
    assert abs(e0[0] - e0[1]) <= 1e-5 * abs(e0[0])
