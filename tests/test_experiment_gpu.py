"""§8(f) row 3: the experiment harness on the device against the reference's
own run_experiment / experiment_csv (zero-timings CSV) and the reference's
named generators (generators.cpp:50-116)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,dims,exact", [("exp", (30, 30, 30), True), ("arcsin", (20, 20, 20, 20), True),
                                             ("tan", (10, 10, 10, 10, 10), False),
                                             ("gaussian", (10, 12, 14), False), ("exp", (7, 9), True)])
def test_named_generators_match_reference(gpu_ctx, ref, name, dims, exact):
    from paper_2403_01778_b200 import experiment as ex
    t = ex.make_tensor(ex.ExperimentSpec(generator=name, dims=list(dims), tensor_seed=5))
    got = t.to_host()
    want = ref.generate(name, dims, 5)
    if exact:
        assert np.array_equal(got, want)
    else:  # device tan / log / cos: last-ulp differences
        assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)) <= 1e-13
        assert np.mean(got == want) > 0.5


def test_experiment_csv_matches_reference(gpu_ctx, ref):
    from paper_2403_01778_b200 import experiment as ex
    dims = (30, 30, 30)
    spec = ex.ExperimentSpec(generator="exp", dims=list(dims), seeds=3, algorithms=["hoscf", "ihoscf"])
    res = ex.run_experiment(spec)
    mine = ex.experiment_csv(res.rows, True).splitlines()
    want_csv, want_table = ref.experiment_csv("exp", ref.generate("exp", dims), dims, ["hoscf", "ihoscf"], 3)
    want = want_csv.splitlines()
    assert mine[0] == want[0] and len(mine) == len(want)
    for m, w in zip(mine[1:], want[1:]):
        mf, wf = m.split(","), w.split(",")
        assert mf[:4] == wf[:4] and mf[7:] == wf[7:]
        assert abs(float(mf[4]) - float(wf[4])) <= 1e-9 * abs(float(wf[4]))
        assert abs(float(mf[5]) - float(wf[5])) <= 1e-9 * abs(float(wf[5]))
        assert abs(int(mf[6]) - int(wf[6])) <= 1
    assert ex.summary_table(res.summaries).splitlines()[0] == want_table.splitlines()[0]
    # phase columns come from the device events
    assert all(r.phase_j_s > 0 and r.phase_eig_s > 0 for r in res.rows)


def test_scaling_and_file_generator(gpu_ctx, oracle, tmp_path):
    import paper_2403_01778_b200 as r1
    from paper_2403_01778_b200 import experiment as ex
    dims = (12, 10, 8)
    a = oracle.oracle_random_tensor(dims, 4)
    p = tmp_path / "a.dt1"
    r1.write_dt1(p, r1.DenseTensor(dims, a))
    spec = ex.ExperimentSpec(generator="file", input_path=str(p), threads=[1, 2], scaling_iters=5)
    rows = ex.run_scaling(spec)
    assert [r.iters for r in rows] == [5, 5] and rows[1].lambda_dev_vs_first == 0.0
    text = ex.scaling_csv(rows).splitlines()
    assert text[0].startswith("generator,dims,algo,threads,iters") and text[1].startswith("file,12x10x8,hoscf,1,5,")
