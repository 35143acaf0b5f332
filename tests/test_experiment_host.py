"""CPU-suite checks of the experiment harness's host logic (formats of
experiment.cpp:48-233: dims text, CSV rows, summary table)."""
import pytest


def test_dims_text_roundtrip():
    from paper_2403_01778_b200 import experiment as ex
    assert ex.format_dims([30, 30, 30]) == "30x30x30"
    assert ex.parse_dims("4x5x6") == [4, 5, 6] and ex.parse_dims("4,5,6") == [4, 5, 6]
    with pytest.raises(ValueError, match="dims must be >= 1"):
        ex.parse_dims("4x0")
    with pytest.raises(ValueError, match="empty dims"):
        ex.parse_dims("x")


def test_csv_and_summary_formats():
    from paper_2403_01778_b200 import experiment as ex
    rows = [ex.RunRow("exp", "30x30x30", "hoscf", 0, 35.49440363123, 0.82069066071, 9, True,
                      0.0123456, 0.0011111, 0.0022222)]
    assert ex.experiment_csv(rows, True) == (
        "generator,dims,algo,seed,lambda,rho,iters,converged,wall_s,phase_j_s,phase_eig_s\n"
        "exp,30x30x30,hoscf,0,35.49440363,0.8206906607,9,1,0,0,0\n")
    assert ex.experiment_csv(rows, False).splitlines()[1].endswith(",0.0123,0.00111,0.00222")
    s = ex.AlgoSummary("hoscf", 3, 3, 35.4944, 0.0, 0.8207, 0.0, 9.6667, 0.5774)
    assert ex.summary_table([s]).splitlines()[1] == \
        "hoscf          35.4944 +- 0.0000   0.8207 +- 0.0000     9.67 +- 0.58   3/3"
    sc = ex.ScalingRow("gaussian", "10x10x10", 1, 10, 0.001, 0.002, 0.0005, 0.2857, 3.5, 0.0)
    assert ex.scaling_csv([sc]).splitlines()[1] == \
        "gaussian,10x10x10,hoscf,1,10,0.001,0.002,0.0005,0.2857,3.5,0"
