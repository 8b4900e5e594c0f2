"""End-to-end comparison: the drop-in pipeline vs the reference pipeline
(rewritten text byte-for-byte, report lines, raised errors)."""
from __future__ import annotations


def outcome(load, transform, text, name, **kw):
    from dartomp.report import plan_lines
    try:
        a = load(path=name, text=text, **({"summary_runner": kw["summary_runner"]}
                                          if "summary_runner" in kw else {}))
    except Exception as e:
        return ("load-error", type(e).__name__, str(e))
    try:
        tkw = {"replay_runner": kw["replay_runner"]} if "replay_runner" in kw else {}
        result, plans = transform(a, **tkw)
    except Exception as e:
        return ("error", type(e).__name__, e.render() if hasattr(e, "render") else str(e))
    try:
        lines = plan_lines(a.src, plans)
    except KeyError as e:      # report.py:35 (no AFTER key) -- same in both
        lines = ["<KeyError %s>" % e]
    return ("ok", result.text, lines)


def compare(text, name, **kw):
    from dartomp.pipeline import load as rload, transform as rtransform
    from paper_2406_13881_b200.pipeline import load, transform
    ref = outcome(rload, rtransform, text, name)
    got = outcome(load, transform, text, name, **kw)
    assert got == ref, "%s: %s" % (name, (ref[:2], got[:2]))
