"""Developer diff: tools/devhost (device pipeline compiled for host) vs the
oracle on the reference corpus, nests and synthetic listings.  Not a test."""
import subprocess
import sys

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402


def dev(listing: bytes, extra=()):
    p = subprocess.run(["build/devhost", *extra], input=listing, capture_output=True, timeout=60)
    if p.returncode != 0:
        return None, p.stderr.decode()[-2000:]
    out = p.stdout
    i = out.rindex(b"\nC ") + 1 if not out.startswith(b"C ") else 0
    # parse trailing C record
    nl = out.index(b"\n", i)
    n = int(out[i + 2:nl])
    return out[nl + 1:nl + 1 + n], out[:i]


def check(name, listing, verbose=True, extra=()):
    ref = O.decompile(listing, fold_local_size="--fold-local-size" in extra)
    got, meta = dev(listing, extra)
    if got is None:
        print(f"CRASH {name}: {meta}")
        return False
    if got != ref.combined:
        if verbose:
            print(f"DIFF {name}")
            print("--- ref\n" + ref.combined.decode(errors="replace"))
            print("--- got\n" + got.decode(errors="replace"))
        return False
    return True


if __name__ == "__main__":
    ok = bad = 0
    if check("copy.asm", open("/root/reference/proj/tests/data/copy.asm", "rb").read()):
        ok += 1
    else:
        bad += 1
    for nm, ls, _, _ in O.corpus():
        if check(nm.decode(), ls):
            ok += 1
        else:
            bad += 1
    shown = 0
    for seed in range(1, int(sys.argv[1]) if len(sys.argv) > 1 else 200):
        r = check(f"nest{seed}", O.make_nest(seed), verbose=shown < 3)
        if r:
            ok += 1
        else:
            bad += 1
            shown += 1
    print("ok", ok, "bad", bad)


def gen(shape, stress, seed, k0, n):
    return subprocess.run(["build/devgen", str(shape), str(stress), str(seed), str(k0), str(n)],
                          capture_output=True, check=True).stdout


def split_kernels(listing: bytes):
    parts = listing.split(b".kernel ")
    return [b".kernel " + p for p in parts[1:]]


def gencmp(shape, stress, seed, n, per=1):
    bad = 0
    for k0 in range(0, n, per):
        ls = gen(shape, stress, seed, k0, per)
        if not check(f"gen{shape}/{stress}/{k0}", ls, verbose=bad < 2):
            bad += 1
    return bad
