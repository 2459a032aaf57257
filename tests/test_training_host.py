"""Host-side training contracts (training.py:36-121, 163-170): sample/spec/config
validation and the random augmentation stream, against the reference's golden
dataset (tests/golden/training_n9.npz).  No GPU."""

import numpy as np
import pytest

from conftest import golden


def test_random_augmentation_is_the_reference_stream():
    from paper_2505_08491_b200 import training as T
    g = golden("training_n9")
    for i in range(5):
        vecs = T.augment_random(9 ** 3, 4, seed=0 * 100_003 + i)
        assert np.array_equal(np.stack(vecs), g["samples"][i, 1:])


def test_validation_errors():
    from paper_2505_08491_b200 import training as T
    with pytest.raises(ValueError, match="unit sphere"):
        T.TrainingSample(np.ones(3), "random", 0)
    with pytest.raises(ValueError, match="unknown sample tag"):
        T.TrainingSample(np.array([1.0, 0.0]), "bogus", 0)
    with pytest.raises(ValueError, match="augmentation mode"):
        T.AugmentationSpec("bogus")
    with pytest.raises(ValueError, match="alpha"):
        T.TrainConfig(epochs=1, alpha=0.0)
    e = T.TrainingDivergedError(7)
    assert e.batch_id == 7 and "batch 7" in str(e)


def test_dataset_split():
    from paper_2505_08491_b200 import training as T
    d = T.Dataset(None, None, [T.GraphRecord(None, None, None, [i]) for i in range(5)], (0, 1, 2, 3), (4,),
                  T.AugmentationSpec())
    assert d.train_samples() == [(0, 0), (1, 1), (2, 2), (3, 3)] and d.val_samples() == [(4, 4)]
