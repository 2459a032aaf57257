"""Dataset construction and FP64 training on the device vs the reference
(tests/golden/training_n9.npz, made by the reference's own build_dataset / train
on its tests' small dataset: 5 family graphs at n = 9, training.py:124-287)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def ds(tmp_path_factory):
    from paper_2505_08491_b200 import assembly as A, geometry as G, training as T
    g = golden("training_n9")
    d = tmp_path_factory.mktemp("graphs")
    graphs = []
    for i in range(5):
        (d / f"g{i}.json").write_bytes(g[f"graph{i}"].tobytes())
        graphs.append(G.load_graph(d / f"g{i}.json"))
    return T.build_dataset(G.StructuredGrid(9), graphs, A.PhysicalParams(), T.AugmentationSpec("random", 4),
                           val_fraction=0.2, seed=0), graphs


def test_dataset_matches_reference(gpu, ds):
    dset, _ = ds
    g = golden("training_n9")
    assert dset.train_indices == tuple(g["train_indices"]) and dset.val_indices == tuple(g["val_indices"])
    for i, rec in enumerate(dset.records):
        assert [s.tag for s in rec.samples] == list(g["tags"][i])
        V = np.stack([s.vector for s in rec.samples])
        assert rel(V[0], g["samples"][i, 0]) <= 1e-9       # physics sample: ILU-FGMRES 1D solve to 1e-4
        assert np.array_equal(V[1:], g["samples"][i, 1:])   # random augmentation: the same numpy stream


def test_alpha_risk_rhs_krylov(gpu, ds):
    from paper_2505_08491_b200 import assembly as A, geometry as G, neural, training as T
    dset, graphs = ds
    g = golden("training_n9")
    alpha = T.compute_alpha(dset)
    assert abs(alpha - float(g["alpha"])) <= 1e-12 * abs(float(g["alpha"]))
    r = T.risk(neural.init_unet_params(1), dset, dset.train_samples(), alpha)
    assert abs(r - float(g["risk_init1"])) <= 1e-10 * abs(float(g["risk_init1"]))
    s0 = A.assemble_coupled_system(G.StructuredGrid(9), graphs[0], A.PhysicalParams())
    b0 = T.generate_rhs(s0)
    assert rel(b0, g["rhs0"]) <= 1e-9
    K = np.stack(T.augment_krylov(A.reduced_operator(s0), b0, 4, 5))
    assert rel(K, g["krylov0"]) <= 1e-7


def test_train_follows_reference(gpu, ds):
    from paper_2505_08491_b200 import training as T
    dset, _ = ds
    g = golden("training_n9")
    p, hist = T.train(dset, T.TrainConfig(epochs=2, seed=0))
    assert len(hist) == 2 and hist[-1][0] < hist[0][0]
    assert rel(np.array(hist), g["history"]) <= 1e-9
    arrays = dict(p.arrays())
    for key, arr in arrays.items():
        ref = g[f"sum:{key}"]
        assert abs(arr.sum() - ref[0]) <= 1e-8 * max(abs(ref[0]), np.sqrt(ref[1])), key
        assert abs((arr * arr).sum() - ref[1]) <= 1e-9 * ref[1], key
    for key in ("head2.kernel", "head2.bias", "head1.bias", "enc1a.bias", "dec1.bias"):
        assert rel(arrays[key], g[f"p:{key}"]) <= 1e-8, key


def test_zero_epochs_and_divergence(gpu, ds):
    from paper_2505_08491_b200 import neural, training as T
    dset, _ = ds
    p, hist = T.train(dset, T.TrainConfig(epochs=0, seed=3))
    assert hist == []
    for (_, a), (_, b) in zip(p.arrays(), neural.init_unet_params(3).arrays()):
        assert np.array_equal(a, b)
    with pytest.raises(T.TrainingDivergedError, match="batch"):
        T.train(dset, T.TrainConfig(epochs=4, learning_rate=1e14, seed=0))


def test_dataset_directory_round_trip(gpu, ds, tmp_path):
    from paper_2505_08491_b200 import training as T
    dset, _ = ds
    T.save_dataset(dset, tmp_path / "d")
    back = T.load_dataset(tmp_path / "d")
    assert back.train_indices == dset.train_indices and back.augmentation == dset.augmentation
    for a, b in zip(dset.records, back.records):
        assert np.array_equal(a.dfield.values, b.dfield.values)
        assert all(np.array_equal(x.vector, y.vector) and x.tag == y.tag for x, y in zip(a.samples, b.samples))
    assert T.compute_alpha(back) == T.compute_alpha(dset)


def test_krylov_augmented_dataset(gpu, ds):
    """AugmentationSpec("krylov", 3, 2): Arnoldi vectors q_2..q_4 of span(b, Cb, ...) on the device
    (training.py:139-160) against the reference's dataset."""
    from paper_2505_08491_b200 import assembly as A, geometry as G, training as T
    _, graphs = ds
    g = golden("training_n9")
    dk = T.build_dataset(G.StructuredGrid(9), graphs[:2], A.PhysicalParams(), T.AugmentationSpec("krylov", 3, 2),
                         val_fraction=0.5, seed=4)
    for i, rec in enumerate(dk.records):
        assert [s.tag for s in rec.samples] == ["physics", "krylov", "krylov", "krylov"]
        for v, ref in zip([s.vector for s in rec.samples], g["krylov_samples"][i]):
            assert rel(v, ref) <= 1e-8
