"""Interchange formats either side of the hot path, pinned to files the reference
wrote (tests/golden/formats_n9.npz, make_golden.py gen_formats): graph JSON
(geometry.py:306-324), MDF1 grid vectors / distance fields (geometry.py:327-363),
MDS1 sample files (training.py:361-393).  MDU3 checkpoints: test_oracle_golden."""

import numpy as np
import pytest

from conftest import golden


def test_graph_json_bytes_and_roundtrip(tmp_path):
    from paper_2505_08491_b200 import geometry as G
    g = golden("formats_n9")
    graph = G.Graph1D(g["vertices"], g["edges"], float(g["radius"]), tuple(int(d) for d in g["dirichlet"]))
    G.save_graph(graph, tmp_path / "g.json")
    assert (tmp_path / "g.json").read_bytes() == g["graph_json"].tobytes()
    (tmp_path / "ref.json").write_bytes(g["graph_json"].tobytes())
    back = G.load_graph(tmp_path / "ref.json")
    assert np.array_equal(back.vertices, graph.vertices) and np.array_equal(back.edges, graph.edges)
    assert back.radius == graph.radius and back.dirichlet_vertices == graph.dirichlet_vertices


def test_mdf1_bytes_and_errors(tmp_path):
    from paper_2505_08491_b200 import geometry as G
    g = golden("formats_n9")
    d = G.DistanceField(G.StructuredGrid(9), g["dvalues"])
    G.save_distance_field(d, tmp_path / "d.bin")
    assert (tmp_path / "d.bin").read_bytes() == g["mdf1"].tobytes()
    (tmp_path / "ref.bin").write_bytes(g["mdf1"].tobytes())
    back = G.load_distance_field(tmp_path / "ref.bin")
    assert back.grid.n == 9 and np.array_equal(back.values, g["dvalues"])
    (tmp_path / "bad.bin").write_bytes(b"XXXX" + g["mdf1"].tobytes()[4:])
    with pytest.raises(ValueError):
        G.read_grid_vector(tmp_path / "bad.bin")
    (tmp_path / "short.bin").write_bytes(g["mdf1"].tobytes()[:-8])
    with pytest.raises(ValueError):
        G.read_grid_vector(tmp_path / "short.bin")
    with pytest.raises(ValueError):
        G.write_grid_vector(tmp_path / "x.bin", 9, np.zeros(10))


def test_mds1_bytes_and_errors(tmp_path):
    from paper_2505_08491_b200 import training as T
    g = golden("formats_n9")
    tags = [str(t) for t in g["tags"]]
    T.write_samples(tmp_path / "s.bin", g["vecs"], tags)
    assert (tmp_path / "s.bin").read_bytes() == g["mds1"].tobytes()
    (tmp_path / "ref.bin").write_bytes(g["mds1"].tobytes())
    vecs, back_tags = T.read_samples(tmp_path / "ref.bin")
    assert np.array_equal(vecs, g["vecs"]) and back_tags == tags
    (tmp_path / "bad.bin").write_bytes(b"MDSX" + g["mds1"].tobytes()[4:])
    with pytest.raises(ValueError):
        T.read_samples(tmp_path / "bad.bin")
    (tmp_path / "short.bin").write_bytes(g["mds1"].tobytes()[:-8])
    with pytest.raises(ValueError):
        T.read_samples(tmp_path / "short.bin")
