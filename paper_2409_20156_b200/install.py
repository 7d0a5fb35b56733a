"""Bind the B200 path into a running reference (xcmix) process.

Rebinds the module globals the reference resolves at call time (SURVEY.md
§8(b)):
  xcmix.anns.retrieve_hard_negatives           <- anns.retrieve_hard_negatives
        (trainer.py:453 and sampler.py:203 call it through the module)
  xcmix.trainer._batch_forward_backward        <- trainer._batch_forward_backward
        (resolved by train_epoch, trainer.py:487)
  xcmix.trainer._assemble_batch_slates         <- trainer._assemble_batch_slates
        (slates="philox"; slates="reference" keeps the reference's PCG64 slates
        so the GPU step can be compared bit-for-bit on identical indices)
  xcmix.trainer/classifiers.apply_classifier_updates_arrays <- classifiers.*
        (trainer.py:27 imported the name, classifiers.py:71 uses the global)
  xcmix.anns.query_topk                        <- anns.query_topk
        (UpToDateHard, trainer.py:321-333; evaluation's anns mode)
  xcmix.evaluation.predict_topk / evaluate     <- evaluation.* (exact mode: batched MIPS)
  xcmix.trainer._uptodate_hard_batch           <- trainer._uptodate_hard_batch (UpToDateHard,
        trainer.py:321-333: one batched MIPS launch vs the live device W)
  xcmix.trainer._probe_full_loss / _eval_p_at  <- trainer.* (the dense per-epoch
        probes, trainer.py:398-423, resolved by train_epoch and the full-loss arm)
  xcmix.trainer.train_full_loss_baseline       <- trainer.train_full_loss_baseline
        (the all-negatives arm, trainer.py:563-616)
Code that imported a name before install() (`from xcmix.anns import f`) keeps
the old object: install first (e.g. from a pytest plugin / conftest).
"""

from __future__ import annotations

from . import _backend, anns, classifiers, evaluation, trainer

_saved: dict = {}


def install(backend=None, slates: str = "philox", fast_step: bool | None = None) -> None:
    """fast_step=True: the drop-in's classifier step takes the single
    label-major pass (grad_emb summed in arrival order: not bitwise
    run-to-run reproducible); default: the deterministic schedule."""
    import xcmix.anns as xa
    import xcmix.classifiers as xc
    import xcmix.trainer as xt

    if fast_step is not None:
        trainer.FAST_STEP = bool(fast_step)
    if slates not in ("philox", "reference"):
        raise ValueError("slates must be 'philox' or 'reference'")
    if backend is not None:
        _backend.set_backend(backend)
    try:
        import xcmix.evaluation as xe
    except ImportError:  # evaluation needs the reference's optional deps
        xe = None
    if not _saved:
        if xe is not None:
            _saved[(xe, "predict_topk")] = xe.predict_topk
            _saved[(xe, "evaluate")] = xe.evaluate
        _saved.update({
            (xa, "query_topk"): xa.query_topk,
            (xa, "retrieve_hard_negatives"): xa.retrieve_hard_negatives,
            (xt, "_batch_forward_backward"): xt._batch_forward_backward,
            (xt, "_uptodate_hard_batch"): xt._uptodate_hard_batch,
            (xt, "_assemble_batch_slates"): xt._assemble_batch_slates,
            (xt, "apply_classifier_updates_arrays"): xt.apply_classifier_updates_arrays,
            (xt, "_probe_full_loss"): xt._probe_full_loss,
            (xt, "_eval_p_at"): xt._eval_p_at,
            (xt, "train_full_loss_baseline"): xt.train_full_loss_baseline,
            (xc, "apply_classifier_updates_arrays"): xc.apply_classifier_updates_arrays,
        })
    anns._approx_impl = _saved[(xa, "retrieve_hard_negatives")]
    anns._approx_query_impl = _saved[(xa, "query_topk")]
    xa.retrieve_hard_negatives = anns.retrieve_hard_negatives
    xa.query_topk = anns.query_topk
    if xe is not None:
        evaluation._reference_predict = _saved[(xe, "predict_topk")]
        evaluation._reference_evaluate = _saved[(xe, "evaluate")]
        xe.predict_topk = evaluation.predict_topk
        xe.evaluate = evaluation.evaluate
    xt._batch_forward_backward = trainer._batch_forward_backward
    xt._uptodate_hard_batch = trainer._uptodate_hard_batch
    xt._assemble_batch_slates = (trainer._assemble_batch_slates if slates == "philox"
                                 else _saved[(xt, "_assemble_batch_slates")])
    xt.apply_classifier_updates_arrays = classifiers.apply_classifier_updates_arrays
    xc.apply_classifier_updates_arrays = classifiers.apply_classifier_updates_arrays
    xt._probe_full_loss = trainer._probe_full_loss
    xt._eval_p_at = trainer._eval_p_at
    xt.train_full_loss_baseline = trainer.train_full_loss_baseline


def uninstall() -> None:
    for (mod, name), fn in _saved.items():
        setattr(mod, name, fn)
    _saved.clear()
    anns._approx_impl = None
    anns._approx_query_impl = None
    evaluation._reference_predict = None
    evaluation._reference_evaluate = None
