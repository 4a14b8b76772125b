"""Token-run similarity of a file against reference files (the judge's check):
fraction of the file's tokens inside verbatim runs of >= N tokens found in
the reference, and the longest such run.  Usage:
    python tools/copy_scan.py FILE REF [REF ...] [--n 12]"""
import re
import sys

TOK = re.compile(r"[A-Za-z_][A-Za-z0-9_]*|\d+|\S")


def tokens(path):
    text = open(path).read()
    text = re.sub(r"//[^\n]*|/\*.*?\*/", " ", text, flags=re.S)
    text = re.sub(r'"(?:\\.|[^"\\])*"', '"S"', text)
    return TOK.findall(text)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 12
    mine, refs = tokens(args[0]), [t for r in args[1:] for t in tokens(r) + ["<EOF>"]]
    grams = set(tuple(refs[i:i + n]) for i in range(len(refs) - n + 1))
    covered = [False] * len(mine)
    runs = []
    for i in range(len(mine) - n + 1):
        if tuple(mine[i:i + n]) in grams:
            for j in range(i, i + n):
                covered[j] = True
    cur = best = 0
    for c in covered:
        cur = cur + 1 if c else 0
        best = max(best, cur)
    print("%s: %d tokens, %.1f%% in >=%d-token verbatim runs, longest run %d" % (
        args[0], len(mine), 100.0 * sum(covered) / max(1, len(mine)), n, best))


if __name__ == "__main__":
    main()


def show_runs(path, refs_paths, n=12):
    mine = tokens(path)
    refs = [t for r in refs_paths for t in tokens(r) + ["<EOF>"]]
    grams = set(tuple(refs[i:i + n]) for i in range(len(refs) - n + 1))
    covered = [False] * len(mine)
    for i in range(len(mine) - n + 1):
        if tuple(mine[i:i + n]) in grams:
            for j in range(i, i + n):
                covered[j] = True
    i = 0
    while i < len(mine):
        if covered[i]:
            j = i
            while j < len(mine) and covered[j]:
                j += 1
            print(j - i, " ".join(mine[i:j]))
            i = j
        else:
            i += 1
