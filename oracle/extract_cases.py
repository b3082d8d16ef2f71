"""TEST INFRASTRUCTURE ONLY: filters one of the reference's doctest files
(/root/reference/proj/tests/*.cpp) down to the test cases whose API the
engine's drop-in headers declare, for the reference-suite build in
oracle/Makefile (target `refsuite`).  The output goes to oracle/_ref/ (git-
ignored build output; nothing from the reference enters the repository).

Everything outside TEST_CASE bodies is kept (includes, helpers), except the
named top-level blocks in --drop (e.g. the `Pipeline` fixture of
test_decomposition.cpp:19-38, which drives the per-batch host tile pipeline
that the engine replaces with the device sweeps).  `#line` directives keep
failure messages pointing at the reference file's own lines.

    python oracle/extract_cases.py SRC OUT --keep-from "counter conformance" \
        --drop "struct Pipeline"
"""
from __future__ import annotations

import argparse
import re


def block_end(text: str, open_brace: int) -> int:
    """Index one past the brace matching text[open_brace] ('{'), skipping
    string/char literals and comments."""
    depth, i, n = 0, open_brace, len(text)
    while i < n:
        c = text[i]
        if c == '"' or c == "'":
            q = c
            i += 1
            while text[i] != q:
                i += 2 if text[i] == "\\" else 1
        elif text.startswith("//", i):
            i = text.index("\n", i)
        elif text.startswith("/*", i):
            i = text.index("*/", i) + 1
        elif c == "{":
            depth += 1
        elif c == "}":
            depth -= 1
            if depth == 0:
                return i + 1
        i += 1
    raise ValueError("unbalanced braces")


def line_of(text: str, pos: int) -> int:
    return text.count("\n", 0, pos) + 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("out")
    ap.add_argument("--keep-from", help="keep test cases from the one with this name on")
    ap.add_argument("--keep", action="append", default=[], help="keep a test case by name")
    ap.add_argument("--drop", action="append", default=[],
                    help="drop the top-level block starting with this text")
    a = ap.parse_args()
    text = open(a.src).read()
    cuts = []  # (begin, end) spans to remove
    for d in a.drop:
        b = text.index(d)
        e = block_end(text, text.index("{", b))
        if text[e:e + 1] == ";":
            e += 1
        cuts.append((b, e))
    keeping = False
    kept = []
    for m in re.finditer(r'TEST_CASE\("((?:[^"\\]|\\.)*)"\)\s*\{', text):
        name = m.group(1)
        e = block_end(text, m.end() - 1)
        if a.keep_from and name == a.keep_from:
            keeping = True
        if keeping or name in a.keep:
            kept.append(name)
        else:
            cuts.append((m.start(), e))
    cuts.sort()
    out, pos = [], 0
    for b, e in cuts:
        out.append(text[pos:b])
        pos = e
        out.append(f'\n#line {line_of(text, e)} "{a.src}"\n')
    out.append(text[pos:])
    with open(a.out, "w") as f:
        f.write(f'#line 1 "{a.src}"\n' + "".join(out))
    print(f"{a.out}: kept {len(kept)} test cases: {kept}")


if __name__ == "__main__":
    main()
