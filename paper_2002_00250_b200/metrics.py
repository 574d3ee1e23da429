"""Segmentation quality metrics with the confusion counts computed on the GPU.

Same names and semantics as the reference module (pkg/src/rgbdseg/
metrics.py:24-101): `ConfusionCounts`, `MetricsReport`, `compare_masks`,
`compute_metrics` (PWC, FNR, FPR, Si; a zero denominator gives None, never 0)
and `aggregate_sequence` (pool the counts over all frames, then derive once).

The counting itself runs on the device, in two forms:
  * `compare_masks(result, gt)` -- one mask against one ground truth
    (rgbdseg_confusion_accumulate);
  * fused into the segmentation kernels: `SegmentationEngine.process_frame(
    frame, labels=gt)` makes K1/K2 count each pixel's decision against the
    label as they write the mask, pooled on the device across frames
    (`engine.confusion_counts()`); `all_reduce_counts` sums such pools over
    the ranks of a multi-GPU run with one NCCL all-reduce.
Labels follow frames.py:27-29: 0 background, 1 foreground, 2 ignore (ignored
pixels count nowhere, metrics.py:50-56).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Optional

GT_BACKGROUND, GT_FOREGROUND, GT_IGNORE = 0, 1, 2  # frames.py:27-29


@dataclass
class ConfusionCounts:
    """metrics.py:24-38."""

    tp: int = 0
    tn: int = 0
    fp: int = 0
    fn: int = 0

    def __add__(self, other: "ConfusionCounts") -> "ConfusionCounts":
        return ConfusionCounts(self.tp + other.tp, self.tn + other.tn, self.fp + other.fp,
                               self.fn + other.fn)

    @property
    def total(self) -> int:
        return self.tp + self.tn + self.fp + self.fn

    @classmethod
    def from_sequence(cls, values) -> "ConfusionCounts":
        tp, tn, fp, fn = (int(v) for v in values)
        return cls(tp, tn, fp, fn)


@dataclass
class MetricsReport:
    """metrics.py:41-47."""

    pwc: Optional[float]
    fnr: Optional[float]
    fpr: Optional[float]
    si: Optional[float]
    counts: ConfusionCounts


def _labels_of(gt):
    return gt.labels if hasattr(gt, "labels") else gt


def compare_masks(result, gt) -> ConfusionCounts:
    """TP/TN/FP/FN between a 0/255 mask and a ground truth (metrics.py:50-69),
    counted on the device.  `gt` is a GroundTruthMask-like object (`.labels`)
    or the (H, W) label array itself; a shape mismatch raises DimensionError."""
    from .frames import confusion_counts

    return ConfusionCounts(*confusion_counts(result, _labels_of(gt)))


def _ratio(num: int, den: int) -> Optional[float]:
    return num / den if den > 0 else None


def compute_metrics(c: ConfusionCounts) -> MetricsReport:
    """PWC = 100(FN + FP)/(TP + FN + FP + TN), FNR = FN/(TP + FN),
    FPR = FP/(FP + TN), Si = TP/(TP + FP + FN) (metrics.py:76-91)."""
    pwc = _ratio(c.fn + c.fp, c.total)
    return MetricsReport(pwc=None if pwc is None else 100.0 * pwc, fnr=_ratio(c.fn, c.tp + c.fn),
                         fpr=_ratio(c.fp, c.fp + c.tn), si=_ratio(c.tp, c.tp + c.fp + c.fn),
                         counts=c)


def aggregate_sequence(per_frame: Iterable[ConfusionCounts]) -> MetricsReport:
    """Pool counts over all frames, then compute the metrics once (metrics.py:94-101)."""
    total = ConfusionCounts()
    seen = False
    for c in per_frame:
        total = total + c
        seen = True
    if not seen:
        raise ValueError("aggregate_sequence needs at least one frame")
    return compute_metrics(total)


def all_reduce_counts(counts, group=None):
    """Sum a device int64[4] (tp, tn, fp, fn) pool over the ranks of a
    torch.distributed group in place (one NCCL all-reduce on GPUs; any
    backend works) and return it as ConfusionCounts."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return ConfusionCounts.from_sequence(counts.tolist())
