"""CPU: the documents point at files that exist -- every `profiles/...`, `tools/...`, `tests/...`, `include/...` path quoted in
DESIGN.md, README.md and profiles/README.md (globs and `…`-abbreviated names aside)."""
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DOCS = ["DESIGN.md", "INTEGRATION.md", "README.md", os.path.join("profiles", "README.md")]
REFERENCE_PATHS = {"tools/sxen_main.cpp"}  # files of the reference (/root/reference/proj), cited as out of scope
PATH = re.compile(r"`((?:profiles|tools|tests|include|oracle|paper_2311_15439_b200)/[A-Za-z0-9_./\-*]+)`")


def test_quoted_paths_exist():
    missing = []
    for doc in DOCS:
        text = open(os.path.join(ROOT, doc), encoding="utf-8").read()
        for m in PATH.finditer(text):
            p = m.group(1).rstrip(".")
            if p.endswith("/") or "_ref" in p or "_build" in p or p.endswith(".so"):
                continue  # directories, built artefacts
            if p in REFERENCE_PATHS:
                continue
            hits = glob.glob(os.path.join(ROOT, p)) if "*" in p else ([p] if os.path.exists(os.path.join(ROOT, p)) else [])
            if not hits:
                missing.append((doc, p))
    assert not missing, missing


def test_profiles_index_lists_every_file():
    index = open(os.path.join(ROOT, "profiles", "README.md"), encoding="utf-8").read()
    unlisted = []
    for name in sorted(os.listdir(os.path.join(ROOT, "profiles"))):
        if name == "README.md":
            continue
        stem = name.rsplit(".", 1)[0]
        # a file is indexed by its name, by a `stem*` / `stem_*` glob, or by a shared prefix written with `_*`
        if name in index or stem in index:
            continue
        prefix_hit = any(g.endswith("*") and name.startswith(g[:-1]) for g in re.findall(r"`([A-Za-z0-9_.\-]+\*)`", index))
        if not prefix_hit:
            unlisted.append(name)
    assert not unlisted, unlisted
