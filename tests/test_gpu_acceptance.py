"""The reference's behavioural acceptance criteria on the device path
(tests/test_acceptance.py:142-197): frames go through apply(rgb, depth16)
(device pack, frames.py:46-88), segmentation, and the device confusion
counts (metrics.compare_masks, metrics.py:50-69)."""

import numpy as np
import pytest

from paper_2002_00250_b200 import synth
from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig

pytestmark = pytest.mark.gpu


def _run_scene(spec, algorithm, mode, gmm=None):
    from paper_2002_00250_b200.engine import SegmentationEngine

    cfg = PipelineConfig(algorithm=algorithm, mode=mode, gmm=gmm or GmmParams(), pbas=PbasParams())
    out = []
    with SegmentationEngine(cfg, spec.width, spec.height, device=0) as eng:
        for t in range(spec.frames):
            rgb, d16, gt = synth.scene_frame(spec, t)
            out.append((eng.apply(rgb, d16 if mode == "rgbd" else None), gt))
    return out


@pytest.mark.parametrize("algorithm", ["gmm", "pbas"])
@pytest.mark.parametrize("mode", ["rgb_only", "rgbd"])
def test_criterion_4_static_burn_in_is_empty(algorithm, mode):
    # tests/test_acceptance.py:142-152: frames 100-119 of a static scene
    spec = synth.SceneSpec("static", frames=120)
    masks = _run_scene(spec, algorithm, mode)
    assert sum(int(m.count_nonzero()) for m, _ in masks[100:120]) == 0


@pytest.mark.parametrize("algorithm", ["gmm", "pbas"])
def test_criterion_5_colour_camouflage_needs_depth(algorithm):
    # tests/test_acceptance.py:164-181: tau = 4 for GMM in both modes;
    # rgb_only Si < 0.1, rgbd Si > 0.9 over the frames with a GT object.
    from paper_2002_00250_b200.frames import confusion_counts

    spec = synth.SceneSpec("colour_camouflage")
    si = {}
    for mode in ("rgb_only", "rgbd"):
        tp = fp = fn = 0
        for mask, gt in _run_scene(spec, algorithm, mode, gmm=GmmParams(tau=4.0)):
            if not gt.any():
                continue
            c = confusion_counts(mask, (gt > 0).astype(np.uint8))
            tp, fp, fn = tp + c[0], fp + c[2], fn + c[3]
        si[mode] = tp / (tp + fp + fn) if tp + fp + fn else 0.0
    assert si["rgb_only"] < 0.1, si
    assert si["rgbd"] > 0.9, si
