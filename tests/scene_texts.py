"""Scene texts shared by the GPU tests and tests/golden/make_golden.py: the
builtin Cornell box at another resolution and/or with a scaled lamp
(the golden generator edits the reference's copy of the same scene the
same way; the packs are sha1-pinned identical, tests/golden/scene_packs.json)."""

import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def edit_scene(text, res, emit_scale=1.0):
    out = []
    for ln in text.splitlines():
        if ln.strip().startswith("resolution"):
            ln = f"resolution {res} {res}"
        elif "camera" in ln and "resolution" in ln:
            head, tail = ln.split("resolution")
            rest = tail.split("}")[1] if "}" in tail else ""
            ln = f"{head}resolution {res} {res} }}{rest}"
        if "emit" in ln and emit_scale != 1.0:
            head, tail = ln.split("emit")
            vals = tail.split("}")[0].split()
            ln = head + "emit " + " ".join(repr(float(v) * emit_scale) for v in vals) + " }"
        out.append(ln)
    return "\n".join(out) + "\n"


def corn_text(res, emit_scale=1.0):
    path = os.path.join(ROOT, "paper_2412_04634_b200", "data", "cornell.scene")
    return edit_scene(open(path).read(), res, emit_scale)
