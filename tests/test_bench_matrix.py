"""The bench harness contract (bench.cpp:139-263) on the B200 side: our CSV
writers produce the reference's bytes — the reference's own load_bench_rows
parses our rows.csv and its writers reproduce rows.csv, summary.csv and
speedup_hist.csv exactly; method tokens parse like parse_method_token."""
import pytest

from paper_2310_00177_b200 import bench_matrix as bm


def test_method_tokens():
    assert bm.parse_method_token("cg") == (True, "cg", "none")
    assert bm.parse_method_token("psdo+neural") == (True, "psdo", "neural")
    assert bm.parse_method_token("pcg+jacobi") == (True, "pcg", "jacobi")
    assert bm.parse_method_token("pcg+foo")[0] is False
    assert bm.parse_method_token("gmres")[0] is False


@pytest.mark.ref
def test_csv_bytes_match_reference_writers(ref, tmp_path):
    rows = []
    for si, system in enumerate(["C1_f000", "C2_f000", "C3_f001"]):
        for mi, m in enumerate(["cg", "pcg+jacobi", "psdo+neural", "fpcg+ic0"]):
            r = bm.BenchRow(system, m, n_f=1000 + si, iterations=10 * (mi + 1) + si, converged=(m != "fpcg+ic0"),
                            setup_seconds=0.001 * (si + 1), iterate_seconds=0.25 / (mi + 1) + 0.01 * si,
                            precond_seconds=0.0, final_rel_residual=9.7e-7 / (mi + 1))
            r.total_seconds = r.setup_seconds + r.iterate_seconds
            if m == "fpcg+ic0":
                r.error = "fpcg+ic0: not available on the B200 device path"
            rows.append(r)
    ours, theirs = tmp_path / "ours", tmp_path / "theirs"
    bm.write_bench_outputs(rows, ours)
    bm.write_bench_report(rows, ours)
    ref.bench_roundtrip(ours / "rows.csv", theirs)
    for name in ("rows.csv", "summary.csv", "speedup_hist.csv"):
        assert (ours / name).read_bytes() == (theirs / name).read_bytes(), name


def test_load_bench_rows_roundtrip(tmp_path):
    """load_bench_rows (bench.cpp:168-201) reads back what write_bench_outputs wrote."""
    rows = [bm.BenchRow("C1", "psdo+neural", n_f=10, iterations=3, converged=True, setup_seconds=0.5,
                        iterate_seconds=0.25, precond_seconds=0.125, total_seconds=0.75, final_rel_residual=1e-7),
            bm.BenchRow("C1", "fpcg+none", error="fpcg+none: not available, on the B200 device path")]
    bm.write_bench_outputs(rows, tmp_path)
    back = bm.load_bench_rows(tmp_path / "rows.csv")
    assert [(r.system, r.method, r.n_f, r.iterations, r.converged, r.total_seconds, r.error) for r in back] == \
           [(r.system, r.method, r.n_f, r.iterations, r.converged, r.total_seconds, r.error) for r in rows]
