"""Training driver over the C-ABI detector: the per-rank loop of the reference's
run_training (src/trainer.cpp:186-283) -- global batch slots, one step, the
rank-0 metrics row, periodic SDCK v1 checkpoints and resume.

metrics.csv (src/trainer.cpp:262-270, 288): header
    step,loss,scale,skipped,step_time_model,peak_bytes
rows "%lld,%.9g,%.9g,%d,%.9g,%lld": the reported (allreduced / K) total loss,
the loss scale USED in the step, 1 when the step overflowed and was skipped,
the step's wall time in ms (the reference writes its analytical model time;
here it is measured), and the device bytes in use.
"""
from __future__ import annotations

import dataclasses
import json
import time
from dataclasses import dataclass, field

from . import ConfigError
from . import detector as D

METRICS_HEADER = "step,loss,scale,skipped,step_time_model,peak_bytes"


def config_digest(p: D.Preset) -> int:
    """64-bit FNV-1a over the canonical JSON of the run's configuration, the
    scheme of the reference's config_digest (src/config.cpp:247-258): the step
    horizon is not part of it (resume may extend it).  The detector preset is
    this driver's config, so the value identifies the same experiment the way
    the reference's does for its own Config."""
    tree = dataclasses.asdict(p)
    s = json.dumps(tree, sort_keys=True, separators=(",", ":"))
    h = 0xCBF29CE484222325
    for ch in s.encode():
        h ^= ch
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def metrics_row(step: int, loss: float, scale: float, skipped: int, step_ms: float, peak: int) -> str:
    return "%d,%.9g,%.9g,%d,%.9g,%d" % (step, loss, scale, skipped, step_ms, peak)


@dataclass
class TrainResult:
    losses: list = field(default_factory=list)
    metrics_csv: str = ""
    skipped: int = 0
    last_step: int = 0


def run_training(p: D.Preset, steps: int, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 metrics_path: str | None = None, checkpoint_path: str | None = None, checkpoint_every: int = 0,
                 resume: str | None = None, force_resume: bool = False) -> TrainResult:
    """train steps (resume.step, steps] with synthetic images and GT keyed by the
    global batch slots (src/dataset.cpp:82-103), so a resumed run sees exactly
    the batches the uninterrupted one would"""
    import torch

    det = D.Detector(p, device=torch.cuda.current_device() if torch.cuda.is_available() else 0, rank=rank,
                     world=world, nccl_id=nccl_id)
    res = TrainResult()
    rows = [METRICS_HEADER]
    start = 0
    digest = config_digest(p)
    if resume:
        start, saved = det.load_checkpoint(resume)
        # the reference refuses a checkpoint of another configuration unless
        # forced (src/trainer.cpp:138-141)
        if saved != digest and not force_resume:
            det.close()
            raise ConfigError(f"checkpoint config digest {saved:#018x} differs from this run's {digest:#018x} "
                                "(pass force_resume=True to override)")
    try:
        for step in range(start + 1, steps + 1):
            t0 = time.perf_counter()
            det.feed(D.batch_slots(step, rank, world, p.batch))
            det.step()
            losses, scale_used, overflow = det.losses()  # synchronises the step
            ms = (time.perf_counter() - t0) * 1e3
            free, total = torch.cuda.mem_get_info()
            res.losses.append(losses[4])
            res.skipped += int(overflow)
            if rank == 0:
                rows.append(metrics_row(step, losses[4], scale_used, int(overflow), ms, total - free))
            if checkpoint_path and checkpoint_every and step % checkpoint_every == 0 and rank == 0:
                det.save_checkpoint(checkpoint_path, step, digest)
            res.last_step = step
    finally:
        det.close()
    res.metrics_csv = "\n".join(rows) + "\n"
    if metrics_path and rank == 0:
        with open(metrics_path, "w") as f:
            f.write(res.metrics_csv)
    return res
