"""Regression text dumps against the live reference's
dump_store_stats / dump_functionals output (tests/golden/make_text_dump_golden.py).

Store statistics are geometry only: byte-identical text.  Functional dumps: keys,
order and sizes identical; checksums (sum(l_g) + sum(l_f)) within relative 1e-12 —
on CPU with the oracle port as the forward map, on the GPU through the device path."""
import json

import numpy as np
import pytest

import paper_1708_02207_b200 as hb
from oracle import hdd_port
from paper_1708_02207_b200 import dumps

from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"

TOL = 1e-12


@pytest.mark.parametrize("level", [4, 5])
def test_store_stats_text(level):
    tree = hb.build_tree(hb.build_mesh(level))
    got = hb.dump_store_stats(hb.store_stats(tree))
    assert got == (GOLDEN / f"dump_store_stats_L{level}.txt").read_text()


def test_store_stats_compressed_refused():
    tree = hb.build_tree(hb.build_mesh(4))
    with pytest.raises(hb.UsageError):
        hb.store_stats(tree, compression=hb.ToleranceSpec(1e-6, 16, 32))


def _problem(f=None):
    meta = json.loads((GOLDEN / "dump_functionals_L5.json").read_text())
    mesh = hb.build_mesh(meta["level"])
    tree = hb.build_tree(mesh)
    obs = tuple((k, int(i)) for k, i in meta["observations"])
    model = hb.MeasurementModel(obs, np.full(len(obs), 0.01), None)
    f = np.ones(mesh.n_nodes) if f is None else f
    return hb.BayesProblem(tree, hb.ParamField.build(tree, 4), f, np.zeros(4 * mesh.n_cells), model), meta


def _parse(text):
    rows = []
    for line in text.strip().split("\n"):
        key, nb, nw, cs = line.split()
        rows.append((key, int(nb), int(nw), float(cs)))
    return rows


def _check(text, k):
    got = _parse(text)
    ref = _parse((GOLDEN / f"dump_functionals_L5_z{k}.txt").read_text())
    assert [r[:3] for r in got] == [r[:3] for r in ref]
    err = max(abs(a[3] - b[3]) / abs(b[3]) for a, b in zip(got, ref))
    assert err <= TOL, err


def _port_forward(problem, Z):
    port = hdd_port.HDDPort(problem.tree.mesh.level, problem.model.observations, f=problem.f)
    return np.stack([port.forward(problem.param.kappa_values(z)) for z in Z])


@pytest.mark.parametrize("k", [0, 1])
def test_dump_functionals_port(k):
    prob, meta = _problem()
    _check(hb.dump_functionals(hb.functional_summaries(prob, meta["z"][k], forward=_port_forward)), k)


def test_dump_functionals_independent_of_f():
    """The checksum is the f = 1 response whatever the problem's own f is."""
    prob, meta = _problem(f=np.linspace(0.0, 2.0, hb.build_mesh(5).n_nodes))
    _check(hb.dump_functionals(hb.functional_summaries(prob, meta["z"][0], forward=_port_forward)), 0)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [0, 1])
def test_dump_functionals_device(k):
    prob, meta = _problem()
    _check(hb.dump_functionals(hb.functional_summaries(prob, meta["z"][k])), k)
    assert dumps.functional_summaries is hb.functional_summaries
