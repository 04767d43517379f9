"""Host-side logic of the B200 path that needs no GPU: configuration errors,
flop model, failure-report ordering, shard balancing."""

import numpy as np
import pytest

from paper_2101_05063_b200 import (ConfigError, InviterConfig, SingularSystemError,
                                   StructuralViolationError, chsrq3in, dhsrq3in, flops, hsrq3in)
from paper_2101_05063_b200.parallel import local_selection, shard_bounds
from paper_2101_05063_b200.solver import raise_first_failure


def test_flop_model_matches_reference_counts():
    # values of hessrq flops.py summed over one solve
    assert flops.per_shift_flops(16000, 128, False) == 653287619
    assert flops.per_shift_flops(16000, 128, True) == 1332957980
    assert flops.per_shift_flops(256, 32, False) == 195254
    assert flops.per_shift_flops(4000, 64, False) == 41683198
    assert abs(flops.reference_flops(16000, 128, 3790, 6105) - 1.0614e13) < 1e10


def test_config_errors_raise_before_any_device_work():
    h = np.triu(np.ones((6, 6)), -1)
    with pytest.raises(ConfigError):
        dhsrq3in(h, [])
    with pytest.raises(ConfigError):
        chsrq3in(h, [1.0 + 0j])
    hr = h.copy()
    hr[3, 2] = 0.0
    with pytest.raises(ConfigError):
        dhsrq3in(hr, [0.5])
    with pytest.raises(ConfigError):
        hsrq3in(h, [0.5, 1 + 1j], InviterConfig(w_max=10))
    with pytest.raises(ConfigError):
        dhsrq3in(h, [0.5], InviterConfig(b_r=7))
    with pytest.raises(ConfigError):
        dhsrq3in(np.ones((5, 5)), [0.5])  # not Hessenberg


def _code(phase, tile, row):
    return (phase << 56) | (tile << 24) | row


def test_first_failure_follows_reference_order():
    codes = np.zeros(10, dtype=np.int64)
    codes[7] = _code(2, 5, 3)   # singular, batch 1 (b_c=4)
    codes[2] = _code(2, 1, 0)   # singular, batch 0, earlier batch wins
    with pytest.raises(SingularSystemError) as e:
        raise_first_failure(codes, 4, [(0, 10)])
    assert e.value.shift_index == 2 and e.value.local_index == 0
    # within a batch: higher tile column first (the sweep runs right to left)
    codes[:] = 0
    codes[1] = _code(2, 3, 9)
    codes[0] = _code(2, 7, 2)
    with pytest.raises(SingularSystemError) as e:
        raise_first_failure(codes, 4, [(0, 10)])
    assert e.value.shift_index == 0
    # any degenerate rotation (reduction phase) precedes every singular pivot
    codes[9] = _code(1, 0, 0)
    with pytest.raises(StructuralViolationError):
        raise_first_failure(codes, 4, [(0, 10)])
    # a failure in the first call (real group) beats one in the second (complex)
    codes[:] = 0
    codes[8] = _code(2, 9, 9)
    codes[1] = _code(2, 0, 0)
    with pytest.raises(SingularSystemError) as e:
        raise_first_failure(codes, 32, [(0, 5), (5, 10)])
    assert e.value.shift_index == 1
    raise_first_failure(np.zeros(4, dtype=np.int64), 4, [(0, 4)])  # no failure: no raise


def test_failure_is_the_references_task_error():
    """A caller of the reference catches the executor's TaskError naming the
    failing graph node, with the kernel's error as cause (scheduler.py:182-187,
    211-214).  Same here -- node kind, coords, seq and message pinned to what
    the live reference raised (golden singular.npz: its dhsrq3 / chsrq3 calls
    and its graph builders) -- and the error is also a SingularSystemError /
    StructuralViolationError instance."""
    from conftest import golden
    from paper_2101_05063_b200 import TaskError
    from paper_2101_05063_b200.core import task_node_of_failure

    g = golden("singular")
    kinds = [str(k) for k in g["node_kinds"]]
    n = 8
    for t in g["tags"]:
        for (b_r, b_c, q, row), node, msg in zip(g[f"{t}_hits"], g[f"{t}_nodes"],
                                                 g[f"{t}_messages"]):
            codes = np.zeros(4, dtype=np.int64)
            codes[q] = _code(2, int(node[1]), int(row))
            with pytest.raises(TaskError) as e:
                raise_first_failure(codes, int(b_c), [(0, 4)], n_tiles=-(-n // int(b_r)))
            err = e.value
            assert isinstance(err, SingularSystemError) and isinstance(err.cause, SingularSystemError)
            assert err.__cause__ is err.cause
            assert (err.shift_index, err.local_index) == (q, row)
            assert (err.cause.shift_index, err.cause.local_index) == (q, row)
            assert err.node.kind == kinds[node[0]]
            assert tuple(err.node.coords) == tuple(int(v) for v in node[1:4])
            assert err.node.seq == node[4]
            assert str(err) == str(msg)
    # node positions in the reference's reduction / substitution graphs
    for N in range(1, 6):
        for b in range(3):
            for tile in range(N):
                assert task_node_of_failure(False, tile, b, N).seq == g["dag_reduce_seq"][N - 1, b, tile]
                nd = task_node_of_failure(True, tile, b, N)
                assert nd.seq == g["dag_solve_seq"][N - 1, b, tile]
                assert nd.kind == ("MergedSolveBacktransform" if tile == 0 else "SolveTile")
    codes = np.zeros(6, dtype=np.int64)
    codes[5] = _code(1, 2, 7)  # degenerate rotation in tile column 2, batch 1 (b_c = 4)
    with pytest.raises(TaskError) as e:
        raise_first_failure(codes, 4, [(0, 6)], n_tiles=3)
    assert isinstance(e.value, StructuralViolationError)
    assert e.value.node.kind == "ReduceDiag" and e.value.node.coords == (2, 2, 1)
    assert str(e.value) == ("task ReduceDiag at (2, 2, 1) failed: degenerate rotation in tile "
                            "column 2 at local row 7, shift 5 (both pivot entries are zero)")


def test_shards_balance_flop_cost():
    rc, cc = shard_bounds(3790, 6105, 8)
    assert rc[0] == cc[0] == 0 and rc[-1] == 3790 and cc[-1] == 6105
    per = [(rc[r + 1] - rc[r]) + 2.04 * (cc[r + 1] - cc[r]) for r in range(8)]
    assert max(per) - min(per) <= 1 + 2.04 + 1e-9
    eigs = np.concatenate([np.arange(5) + 0.5, np.arange(4) + 1j])
    seen = np.concatenate([local_selection(eigs, r, 3)[0] for r in range(3)])
    assert sorted(seen.tolist()) == list(range(9))


def test_task_flops_match_reference_runstats():
    """flops_* / formula_* columns of the bench CSV = the reference's RunStats."""
    from conftest import golden

    g = golden("runstats")
    for t in g["tags"]:
        n, b_r, m, c = (int(v) for v in g[f"{t}_meta"])
        ex, fo = flops.task_flops(n, b_r, m, bool(c))
        assert [ex[k] for k in flops.TASK_TYPES] == list(g[f"{t}_flops"])
        assert [fo[k] for k in flops.TASK_TYPES] == list(g[f"{t}_formula"])


def test_bench_csv_inputs_and_header(tmp_path):
    """Same shifts as the reference bench generator, same leading CSV header."""
    from conftest import golden
    from paper_2101_05063_b200 import HessenbergMatrix, benchcsv

    g = golden("runstats")
    h = HessenbergMatrix(g["shifts_h"])
    assert np.array_equal(benchcsv.gen_shifts(h, 7, "real"), g["shifts_real"])
    assert np.array_equal(benchcsv.gen_shifts(h, 7, "complex"), g["shifts_cplx"])
    ref_head = [str(v) for v in g["bench_header"]]
    assert benchcsv.header()[: len(ref_head)] == ref_head
    with pytest.raises(ConfigError):  # matrix files: out of scope
        benchcsv.load_matrix(str(tmp_path / "m.bin"))


def test_verify_suite_matrices_match_reference_fixtures():
    """gpu_verifysuite.paper_h restates the paper's H2 / H3 (§5.2) exactly: the golden
    solves' gen_h2(60) / gen_h3(60) matrices."""
    from conftest import golden
    from gpu_verifysuite import paper_h

    g = golden("solves")
    hs = {tuple(np.asarray(g[f"{t}_h"]).ravel()[:3]): np.asarray(g[f"{t}_h"]) for t in g["tags"]
          if np.asarray(g[f"{t}_h"]).shape == (60, 60)}
    h2, h3 = paper_h(60, -60).data, paper_h(60, 0.5).data
    assert any(np.array_equal(h, h2) for h in hs.values())
    assert any(np.array_equal(h, h3) for h in hs.values())


def test_api_types_of_the_reference_surface():
    """The types a caller of the reference's path constructs or receives
    (core.py:105-129, 263-300; overflow.py:30-47) exist here with the same
    constructor checks, methods and values."""
    import paper_2101_05063_b200 as P

    g = P.TileGrid(300, 128)
    assert (g.n, g.b_r, g.N, g.ranges) == (300, 128, 3, [(0, 128), (128, 256), (256, 300)])
    assert g.tile_of(255) == 1 and g.tile_slice(2) == slice(256, 300)
    assert repr(g) == "TileGrid(n=300, b_r=128, N=3)"
    with pytest.raises(ConfigError):
        P.TileGrid(10, 11)
    b = P.OverflowBudget.for_grid(g)
    dmax = float(np.finfo(np.float64).max)
    assert b.omega == dmax / 2.0 / 128 and b.safety_divisor == 128
    assert P.OverflowBudget.for_tile_rows(64) == P.OverflowBudget(dmax / 2.0 / 64, 64)
    for bad in (0.0, dmax):
        with pytest.raises(ValueError):
            P.OverflowBudget(bad)
    with pytest.raises(ValueError):
        P.OverflowBudget(dmax / 2.0, 4)
    w = P.Workspace()
    a = w.take("x", (3, 4), crossover=True)
    assert a.shape == (3, 4) and w.peak_crossover_reals == 12
    assert w.take("x", (2, 2)).base is a.base  # reused allocation
    z = np.array([[1 + 2j, 3 - 4j]])
    assert np.array_equal(P.interleave_complex(z), [[1.0, 2.0, 3.0, -4.0]])
    assert np.array_equal(P.deinterleave_complex(P.interleave_complex(z)), z)
    with pytest.raises(ConfigError):
        P.deinterleave_complex(np.zeros((2, 3)))
    h = P.HessenbergMatrix(np.triu(np.arange(16.0).reshape(4, 4), -1))
    assert np.array_equal(h.subdiagonal(), [4.0, 9.0, 14.0]) and h.is_unreduced()


def test_api_surface_matches_installed_reference():
    """With the reference importable (baseline/_ref in the build container):
    every driver accepts the reference's positional / keyword arguments, and the
    config / result types carry at least the reference's fields with the same
    defaults, in the same order."""
    import dataclasses
    import inspect
    import os
    import sys

    from conftest import ROOT

    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "hessrq")):
        pytest.skip("reference not installed under baseline/_ref")
    sys.path.insert(0, ref)
    try:
        import hessrq.backsolve as rb
        import hessrq.core as rc
        import hessrq.inviter as ri
        import hessrq.scheduler as rs
    finally:
        sys.path.remove(ref)
    import paper_2101_05063_b200 as P

    for name, rf in (("hsrq3in", ri.hsrq3in), ("dhsrq3in", ri.dhsrq3in), ("chsrq3in", ri.chsrq3in),
                     ("dhsrq3", rb.dhsrq3), ("chsrq3", rb.chsrq3), ("converged", ri.converged),
                     ("starting_vector", ri.starting_vector)):
        want = list(inspect.signature(rf).parameters.values())
        got = list(inspect.signature(getattr(P, name)).parameters.values())
        assert [(p.name, p.kind, p.default) for p in got[:len(want)]] == \
               [(p.name, p.kind, p.default) for p in want], name
        assert all(p.default is not inspect.Parameter.empty for p in got[len(want):]), name
    for name, mod in (("InviterConfig", ri), ("EigvecResult", ri), ("SolutionBlock", rc)):
        want = dataclasses.fields(getattr(mod, name))
        got = dataclasses.fields(getattr(P, name))
        for fw, fg in zip(want, got):
            assert fw.name == fg.name, (name, fw.name, fg.name)
            if fw.default is not dataclasses.MISSING:
                assert fw.default == fg.default, (name, fw.name)
    for cls in ("HessrqError", "ConfigError", "SingularSystemError", "StructuralViolationError"):
        assert [b.__name__ for b in getattr(P, cls).__mro__] == \
               [b.__name__ for b in getattr(rc, cls).__mro__], cls
    assert [b.__name__ for b in P.TaskError.__mro__] == [b.__name__ for b in rs.TaskError.__mro__]
    for cls, mod in (("TileGrid", rc), ("HessenbergMatrix", rc), ("ScalingMatrix", rc),
                     ("Workspace", rc), ("TaskNode", rs)):
        want = {m for m in dir(getattr(mod, cls)) if not m.startswith("_")}
        got = {m for m in dir(getattr(P, cls)) if not m.startswith("_")}
        assert want <= got, (cls, want - got)


def test_committed_bench_lines_carry_the_contract_keys():
    """The bench lines kept under profiles/ (both arms, last run of the round)
    carry every key of the bench contract with consistent values."""
    import json
    import os

    from conftest import ROOT

    def load(name):
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.loads(f.read().strip().splitlines()[-1])

    d = load("r02g_bench_final.json")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["dtype"] == "f64" and d["higher_is_better"] is True and d["vs_baseline"] is None
    assert "workload" in d["config"] and "model" not in d["config"]
    assert abs(d["value"] - 9895 / (d["ms_per_step"] / 1e3)) < 1e-6 * d["value"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "tensor" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert 0.9 < r["traffic"] / r["traffic_detail"]["algorithmic_bytes"] < 1.1
    c = d["cpu_baseline"]
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1 and "sample" in c
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 2e9 and e["d2h_bytes_per_step"] > 2e9
    assert e["value"] < d["value"]  # the transfers are inside the timed region
    assert d["gpu_launches"] > 0 and d["clocks"]["reasons"] == []
    ref = load("r02f_bench_reference_arm.json")
    assert ref["impl"] == "reference" and ref["config"] == d["config"]
    assert ref["metric"] == d["metric"] and ref["unit"] == d["unit"]
    assert ref["e2e"]["h2d_bytes_per_step"] == 0 and ref["e2e"]["value"] == ref["value"]
