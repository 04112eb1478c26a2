"""Per-decision oracle check of the device dispatcher's decision log."""
import rrfp_oracle as O


def check_decisions(decisions, w, hint, limit, ranked=()):
    """Re-evaluate every logged device decision with the reference's
    update_backpressure + arbitrate (oracle restatement, arbitration.py:188-303)
    on exactly the inputs the device saw."""
    bad = []
    for d in decisions:
        ctl = O.StageCtl(limit, w.num_chunks, w.num_microbatches)
        ctl.nf, ctl.nb = d["n_f"], d["n_b"]
        ctl.mode, ctl.focus = d["mode_in"], d["focus_in"]
        ctl.done = {(mb, c, "F") for mb, c in d["doneF"]} | {(mb, c, "B") for mb, c in d["doneB"]}
        ctl.update_bp()
        ctl.phase = d["phase"]
        v = O.View()
        v.fready, v.bready, v.wpend = set(d["fready"]), set(d["bready"]), set(d["wpend"])
        v.admission = d["admission"] if d["admission"] >= 0 else None
        kind, task = O.arbitrate(v, ctl, hint.kind, w.decompose_backward, ranked)
        if (ctl.mode, ctl.focus) != (d["mode"], d["focus"]) or (kind, task) != (d["kind"], d["task"]):
            bad.append((d, (ctl.mode, ctl.focus, kind, task)))
    return bad
