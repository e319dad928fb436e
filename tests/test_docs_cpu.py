"""The evidence the docs cite exists: every profiles/ path named in DESIGN.md, README.md, INTEGRATION.md and the
kernel sources is in the tree (brace / glob patterns excepted)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DOCS = ["DESIGN.md", "README.md", "INTEGRATION.md", "profiles/README.md"]


def test_cited_profiles_exist():
    missing = []
    for doc in DOCS:
        text = open(os.path.join(ROOT, doc)).read()
        for m in re.finditer(r"profiles/[A-Za-z0-9_./-]+", text):
            path = m.group(0).rstrip(".,)")
            nxt = text[m.end():m.end() + 1]
            if path.endswith("/") or nxt in ("*", "{"):  # a directory, a glob or a brace pattern
                continue
            if not os.path.exists(os.path.join(ROOT, path)):
                missing.append((doc, path))
    assert not missing, missing
