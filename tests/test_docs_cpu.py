"""The evidence the docs cite exists: every file named in backticks in profiles/README.md,
README.md and DESIGN.md that looks like a profiles/, tools/ or tests/ file is in the repo."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cited(md):
    text = open(os.path.join(ROOT, md)).read()
    return set(re.findall(r"`([A-Za-z0-9_./{},*-]+\.(?:json|md|txt|py|cu|sh|csv))`", text))


def _expand(name):
    m = re.search(r"\{([^}]*)\}", name)
    if not m:
        return [name]
    return [p for alt in m.group(1).split(",") for p in _expand(name[:m.start()] + alt + name[m.end():])]


def test_cited_evidence_files_exist():
    missing = []
    for md, base in (("profiles/README.md", "profiles/r02"), ("profiles/r01/README.md", "profiles/r01"),
                     ("README.md", ""), ("DESIGN.md", "")):
        for name in _cited(md):
            if "*" in name or name in ("SPEC.md", "PAPER.md"):   # the reference's own documents
                continue
            for n in _expand(name):
                dirs = ("", base, "profiles", "profiles/r01", "profiles/r01/history", "profiles/r02", "profiles/r02final", "tools", "tests",
                        "include", "oracle", "aa_inputs", "paper_2110_09667_b200", "paper_2110_09667_b200/csrc")
                candidates = [os.path.join(ROOT, d, n) for d in dirs]
                if not any(os.path.exists(c) for c in candidates):
                    missing.append((md, n))
    assert not missing, missing
