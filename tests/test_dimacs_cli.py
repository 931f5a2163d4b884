"""DIMACS ingest, the seeded generator and the CLI.

Mirrors the reference's tests/test_io_cli.py: the same samples, mutations and
error messages, byte-exact round trips, and the generator pinned to the reference's
fixture files through their sha256 (tests/golden/fixture_hashes.json, written by
tests/golden/make_fixture_hashes.py from /root/reference).  Parsing runs in the
C++ part of libfm_b200.so and needs no GPU; solving through the CLI does."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import ROOT, grid_caps

from paper_1110_6231_b200 import (
    GridNetwork,
    ParseError,
    cli_main,
    detect_kind,
    generate,
    load_max,
    parse_dimacs_asn,
    parse_dimacs_max,
    serialize_instance,
    serialize_network,
)
from paper_1110_6231_b200 import generators as G

MAX_SAMPLE = """\
p max 4 5
n 1 s
n 4 t
a 1 2 3
a 1 3 2
a 2 4 2
a 3 4 3
a 2 3 1
"""

ASN_SAMPLE = """\
p asn 4 3
n 1
n 2
a 1 3 5
a 2 3 1
a 2 4 7
"""

with open(os.path.join(ROOT, "tests", "golden", "fixture_hashes.json")) as _f:
    FIXTURES = json.load(_f)


def fixture_text(name):
    kind, n, m_or_density, max_value, seed = FIXTURES[name]["generate"]
    return generate(kind, n, m_or_density, max_value, seed).to_text()


@pytest.mark.parametrize("name", sorted(FIXTURES))
def test_generator_reproduces_reference_fixtures(name):
    text = fixture_text(name)
    assert len(text.encode()) == FIXTURES[name]["bytes"]
    assert hashlib.sha256(text.encode()).hexdigest() == FIXTURES[name]["sha256"]


def test_parse_max_sample():
    net = parse_dimacs_max(MAX_SAMPLE)
    assert net.node_count == 4
    assert net.source == 0 and net.sink == 3
    assert net.arc_count == 10
    assert net.capacity[0] == 3
    assert net.tail[1] == 1 and net.head[1] == 0 and net.capacity[1] == 0
    assert net.out_arcs[1] == [1, 4, 8]


def test_parse_max_accepts_comments_and_blank_lines():
    assert parse_dimacs_max("c header comment\n\nc another\n" + MAX_SAMPLE).node_count == 4


def test_serialize_round_trips_are_byte_exact():
    assert serialize_network(parse_dimacs_max(MAX_SAMPLE)) == MAX_SAMPLE
    inst = parse_dimacs_asn(ASN_SAMPLE)
    assert inst.n == 2 and inst.edges == ((0, 0, 5), (1, 0, 1), (1, 1, 7)) and not inst.complete
    assert serialize_instance(inst) == ASN_SAMPLE
    assert parse_dimacs_asn(ASN_SAMPLE.replace("a 2 4 7", "a 4 2 7")) == inst
    for name in FIXTURES:
        text = fixture_text(name)
        if name.endswith(".max"):
            assert serialize_network(parse_dimacs_max(text)) == text
        else:
            assert serialize_instance(parse_dimacs_asn(text)) == text


@pytest.mark.parametrize(
    "mutation, message",
    [
        (lambda t: "p max 4 5\n" + t, "line 2: duplicate problem line"),
        (lambda t: "n 1 s\n" + t, "line 1: 'n' line before problem line"),
        (lambda t: t.replace("n 1 s", "n 1"), "line 2: malformed node designator"),
        (lambda t: t.replace("n 4 t", "n 4 s"), "line 3: duplicate source designator"),
        (lambda t: t.replace("n 4 t", "n 4 x"), "line 3: node designator must be 's' or 't'"),
        (lambda t: t.replace("n 4 t", "n 1 t"), "line 3: source and sink are the same"),
        (lambda t: t.replace("a 1 2 3", "a 1 2"), "line 4: malformed arc line"),
        (lambda t: t.replace("a 1 2 3", "a 1 2 -3"), "line 4: negative capacity"),
        (lambda t: t.replace("a 1 2 3", "a 1 9 3"), "line 4: node id 9 out of range"),
        (lambda t: t.replace("a 1 2 3", "q 1 2 3"), "line 4: unrecognized line type"),
        (lambda t: t.replace("a 2 3 1\n", ""), "arc count mismatch"),
        (lambda t: t.replace("p max", "p asn"), "expected problem type 'max'"),
        (lambda t: t.replace("a 1 2 3", "a 1 2 x"), "expected integer, got 'x'"),
    ],
)
def test_parse_max_error_messages(mutation, message):
    with pytest.raises(ParseError, match=message):
        parse_dimacs_max(mutation(MAX_SAMPLE))


def test_parse_max_missing_pieces():
    with pytest.raises(ParseError, match="missing problem line"):
        parse_dimacs_max("c empty\n")
    with pytest.raises(ParseError, match="missing source designator"):
        parse_dimacs_max("p max 2 0\nn 2 t\n")
    with pytest.raises(ParseError, match="missing sink designator"):
        parse_dimacs_max("p max 2 0\nn 1 s\n")


@pytest.mark.parametrize(
    "mutation, message",
    [
        (lambda t: t.replace("n 2\n", ""), "sides must be the same size"),
        (lambda t: t.replace("a 1 3 5", "a 1 2 5"), "edge endpoints on the same side"),
        (lambda t: t.replace("a 2 4 7\n", ""), "edge count mismatch"),
        (lambda t: t.replace("n 1\n", "n\n"), "line 2: malformed node designator"),
        (lambda t: t.replace("p asn", "p max"), "expected problem type 'asn'"),
    ],
)
def test_parse_asn_error_messages(mutation, message):
    with pytest.raises(ParseError, match=message):
        parse_dimacs_asn(mutation(ASN_SAMPLE))


def test_detect_kind():
    assert detect_kind(MAX_SAMPLE) == "maxflow"
    assert detect_kind(ASN_SAMPLE) == "assignment"
    with pytest.raises(ParseError, match="missing problem line"):
        detect_kind("c nothing here\n")


def test_generate_validation_and_determinism():
    assert generate("maxflow", 10, 20, 30, 4).to_text() == generate("maxflow", 10, 20, 30, 4).to_text()
    assert generate("maxflow", 10, 20, 30, 4).to_text() != generate("maxflow", 10, 20, 30, 5).to_text()
    with pytest.raises(ValueError, match="n >= 2"):
        generate("maxflow", 1, 1)
    with pytest.raises(ValueError, match="arc count m >= 1"):
        generate("maxflow", 3, 0)
    with pytest.raises(ValueError, match="density"):
        generate("assignment", 3, 1.5)
    with pytest.raises(ValueError, match="unknown kind"):
        generate("mincost", 3, 1)


@pytest.mark.parametrize("H,W,kind", [(5, 7, "G"), (1, 9, "G"), (9, 1, "S"), (16, 12, "S")])
def test_grid_file_is_detected_and_planes_round_trip(H, W, kind):
    caps = grid_caps({"H": H, "W": W, "seed": 3, "kind": kind})
    net = GridNetwork(*caps)
    text = serialize_network(net)
    got, extra = load_max(text)
    assert extra == 0 and isinstance(got, GridNetwork)
    if W > 1 and H > 1:
        assert (got.H, got.W) == (H, W)
    # whatever the inferred layout, the arc multiset of the network is identical
    a = sorted(zip(*[x.tolist() for x in got.arc_arrays()]))
    b = sorted(zip(*[x.tolist() for x in net.arc_arrays()]))
    assert [x for x in a if x[2]] == [x for x in b if x[2]]


def test_non_grid_file_falls_back_to_general_network():
    got, extra = load_max(fixture_text("maxflow_small.max"))
    assert not isinstance(got, GridNetwork) and extra == 0


def test_cli_gen_and_input_errors(tmp_path, capsys):
    path = tmp_path / "inst.max"
    assert cli_main(["gen", "--kind", "maxflow", "--n", "12", "--m", "25", "--max-value", "50",
                     "--seed", "7", "--output", str(path)]) == 0
    assert path.read_text() == fixture_text("maxflow_small.max")
    capsys.readouterr()
    assert cli_main(["maxflow", "--input", "/nonexistent/file.max"]) == 2
    bad = tmp_path / "bad.max"
    bad.write_text(MAX_SAMPLE.replace("a 1 2 3", "a 1 2 -3"))
    assert cli_main(["maxflow", "--input", str(bad)]) == 2
    assert "line 4: negative capacity" in capsys.readouterr().err
    assert cli_main(["frobnicate"]) == 2


def _run(capsys, *argv):
    code = cli_main(list(argv))
    cap = capsys.readouterr()
    return code, cap.out, cap.err


@pytest.mark.gpu
def test_cli_maxflow_and_verify_on_fixtures(tmp_path, capsys, golden):
    values = {c["name"]: c["value"] for c in golden["maxflow"] if c["name"].startswith("fixture")}
    for name in ("maxflow_small.max", "maxflow_medium.max", "maxflow_fixed.max"):
        path = tmp_path / name
        path.write_text(fixture_text(name))
        for extra in ([], ["--mode", "par", "--workers", "2"]):
            code, out, err = _run(capsys, "maxflow", "--input", str(path), *extra)
            assert code == 0, err
            rec = json.loads(out)
            assert rec["objective"] == values[f"fixture {name}"]
            assert set(rec) >= {"objective", "pushes", "relabels", "rounds", "elapsed_ms", "mode", "workers"}
        code, out, err = _run(capsys, "verify", "--input", str(path))
        assert code == 0, err
        assert json.loads(out)["oracle_objective"] == values[f"fixture {name}"]


@pytest.mark.gpu
def test_cli_grid_file_matches_oracle(tmp_path, capsys):
    import oracle

    caps = grid_caps({"H": 40, "W": 56, "seed": 5, "kind": "S"})
    text = serialize_network(GridNetwork(*caps))
    text = text.replace(f"p max {40 * 56 + 2} ", "c grid file\np max %d " % (40 * 56 + 2))
    path = tmp_path / "grid.max"
    path.write_text(text)
    cut_path = tmp_path / "cut.txt"
    code, out, err = _run(capsys, "maxflow", "--input", str(path), "--cut-output", str(cut_path))
    assert code == 0, err
    rec = json.loads(out)
    want = oracle.grid_maxflow(*caps, solver="seq")
    assert rec["objective"] == want["value"] and rec["grid"] == [40, 56]
    cut = np.loadtxt(cut_path, dtype=np.uint8).astype(bool)
    assert (cut == want["cut"].reshape(-1)).all()
    # GPU metrics in the record
    assert rec["launches"] > 0 and rec["device_ms"] > 0 and rec["medges_per_s"] > 0
    assert rec["bfs_levels"] >= 1 and rec["hbm_gbs_achieved"] > 0
    code, out, err = _run(capsys, "verify", "--input", str(path))
    assert code == 0, err
    # --gpus 2: the same grid in two row bands (virtual bands on the one test GPU)
    code, out, err = _run(capsys, "maxflow", "--input", str(path), "--gpus", "2", "--cut-output", str(cut_path))
    assert code == 0, err
    rec = json.loads(out)
    assert rec["objective"] == want["value"] and rec["gpus"] == 2
    assert (np.loadtxt(cut_path, dtype=np.uint8).astype(bool) == want["cut"].reshape(-1)).all()


@pytest.mark.gpu
def test_cli_assign_and_verify(tmp_path, capsys):
    path = tmp_path / "inst.asn"
    path.write_text(fixture_text("assign_complete_n5.asn"))
    for extra in ([], ["--mode", "par", "--workers", "4"], ["--no-heuristics"]):
        code, out, err = _run(capsys, "assign", "--input", str(path), *extra)
        assert code == 0, err
        assert json.loads(out)["objective"] == 410
    code, out, err = _run(capsys, "verify", "--input", str(path))
    assert code == 0, err
    rec = json.loads(out)
    assert rec["objective"] == rec["oracle_objective"] == 410
    for name, want in (("assign_sparse_n6.asn", 366), ("assign_fixed_n8.asn", 695)):
        p = tmp_path / name
        p.write_text(fixture_text(name))
        code, out, err = _run(capsys, "verify", "--input", str(p))
        assert code == 0, err
        assert json.loads(out)["objective"] == want


@pytest.mark.gpu
def test_cli_infeasible_assignment_exits_one(tmp_path, capsys):
    path = tmp_path / "bad.asn"
    path.write_text("p asn 4 2\nn 1\nn 2\na 1 3 5\na 2 3 3\n")
    code, out, err = _run(capsys, "assign", "--input", str(path))
    assert code == 1 and "infeasible" in err
