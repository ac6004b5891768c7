"""Every profile / tool / test file DESIGN.md and the READMEs cite exists in the repository (the
measurements they quote are committed, not described from memory)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cited(path):
    text = open(os.path.join(ROOT, path)).read()
    return set(re.findall(r"`((?:profiles|tools|tests|examples|oracle|include|paper_2103_03330_b200|dgz_inputs)/[\w./-]+)`", text))


def test_design_and_readme_citations_exist():
    missing = []
    for doc in ("DESIGN.md", "README.md", "profiles/r01/README.md", "profiles/r02/README.md", "tools/README.md"):
        for p in _cited(doc):
            full = os.path.join(ROOT, p)
            if not os.path.exists(full):
                missing.append((doc, p))
    assert not missing, missing


def test_profile_readme_lists_files():
    for r in ("r01", "r02"):
        listed = open(os.path.join(ROOT, "profiles", r, "README.md")).read()
        for name in re.findall(r"`([\w.-]+\.(?:jsonl|json|csv|txt))`", listed):
            if "*" in name:
                continue
            assert os.path.exists(os.path.join(ROOT, "profiles", r, name)) or \
                os.path.exists(os.path.join(ROOT, "profiles", name)), name
