"""Randomized differential test of the CUDA path against the oracle (development tool).

    python tools/fuzz.py [seconds=240] [seed=0]

Each case draws an input format, a size (log-uniform up to 2^22), a base misalignment, a content
mix (uniform bit patterns, a narrow exponent band, cancelling pairs, sprinkled NaN/Inf, zeros and
subnormals) and an API (fused sum, chunked accumulate, host streaming, shard merge, sparse image
round trip, equal segments with or without images / CSR segments, checkpoint / resume, strided
reductions, the condition-number-sensitive sum vs oracle/condsens.py), and compares value bits,
binary32 bits, flags and the canonical image with the oracle. Prints one line per failure (with the case seed) and a summary."""
from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1605_05436_b200 as xs  # noqa: E402

FMTS = {"f64": (np.uint64, 52, 11, torch.float64, torch.int64), "f32": (np.uint32, 23, 8, torch.float32, torch.int32),
        "f16": (np.uint16, 10, 5, torch.float16, torch.int16), "bf16": (np.uint16, 7, 8, torch.bfloat16, torch.int16)}


def content(rng, fmt: str, n: int) -> np.ndarray:
    ut, t, l, _, _ = FMTS[fmt]
    bits = 8 * np.dtype(ut).itemsize
    em = ((1 << l) - 1) << t
    raw = rng.integers(0, 1 << 62, size=n, dtype=np.uint64) * np.uint64(4) + rng.integers(0, 4, size=n,
                                                                                          dtype=np.uint64)
    b = (raw & np.uint64((1 << bits) - 1)).astype(ut) if bits < 64 else raw.astype(ut)
    kind = rng.integers(0, 5)
    if kind == 1:                                       # narrow exponent band
        e0 = int(rng.integers(1, (1 << l) - 3))
        e = rng.integers(e0, e0 + 3, size=n).astype(np.uint64)
        b = ((b & ut(~em & ((1 << bits) - 1))) | (e << np.uint64(t)).astype(ut)).astype(ut)
    fin = (b & ut(em)) == ut(em)
    b[fin] ^= ut(1 << t)
    if kind == 2 and n > 1:                             # cancelling pairs
        h = n // 2
        b[h:2 * h] = b[:h] ^ ut(1 << (bits - 1))
    if kind == 3 and n:                                 # zeros, signed zeros, subnormals
        k = rng.integers(0, n, size=max(1, n // 7))
        b[k] = (rng.integers(0, 1 << t, size=k.size).astype(np.uint64) |
                (rng.integers(0, 2, size=k.size).astype(np.uint64) << np.uint64(bits - 1))).astype(ut)
    if rng.random() < 0.3 and n:                        # sprinkled specials
        k = rng.integers(0, n, size=int(rng.integers(1, 4)))
        b[k] = np.array([em, em | (1 << (bits - 1)), em | 1], dtype=np.uint64)[rng.integers(0, 3, size=k.size)] \
            .astype(ut)
    return b


def ref(fmt: str, b: np.ndarray):
    if fmt == "f64":
        return oracle.exact_sum(b.view(np.float64))
    if fmt == "f32":
        return oracle.exact_sum(b.view(np.float32))
    return oracle.exact_sum(b, fmt=fmt)


def to_dev(b: np.ndarray, fmt: str, off: int):
    _, _, _, dt, it = FMTS[fmt]
    buf = torch.empty(b.size + 16, dtype=it, device="cuda")
    t = buf[off:off + b.size]
    t.copy_(torch.from_numpy(b.view(np.dtype(it.__repr__().split(".")[-1]))))
    return t.view(dt)


def same(res, canon, r, limbs) -> bool:
    return (res.bits == r.bits and res.bits_f32 == r.bits_f32 and res.flags == r.flags and
            (canon is None or (np.asarray(canon, dtype=np.uint64) == limbs).all()))


def one_case(seed: int) -> str | None:
    rng = np.random.default_rng(seed)
    fmt = ["f64", "f32", "f16", "bf16"][rng.integers(0, 4)]
    n = int(2 ** rng.uniform(0, 22)) if rng.random() < 0.9 else int(rng.integers(0, 64))
    off = int(rng.integers(0, 8))
    b = content(rng, fmt, n)
    d = to_dev(b, fmt, off)
    api = rng.integers(0, 9)
    if api == 8:                                          # condition-number-sensitive sum (binary64)
        if fmt != "f64" or n > 6000:
            return None
        from oracle import condsens as cs
        rule = int(rng.integers(1, 3))
        res, info, canon = xs.condsens_sum(d, rule)
        vals = b.view(np.float64).tolist()
        o = cs.condsens_sum(vals, rule=rule)
        ok = info.r == o.r and info.iterations == o.iterations and info.exact == o.exact
        if o.r <= 16:
            ok = ok and info.e_cut == o.e_cut and info.root == o.root
        ob = int(np.array([o.value], dtype=np.float64).view(np.uint64)[0])
        ok = ok and (res.bits == ob or (np.isnan(o.value) and np.isnan(res.value)))
        return None if ok else f"f64 n={n} condsens rule {rule}"
    if api == 7 and n:                                    # strided reduction [outer][len][inner]
        inner = int(rng.integers(2, 80))
        outer = int(rng.integers(1, 4))
        length = n // (outer * inner)
        if length == 0:
            return None
        m = outer * length * inner
        o64, o32, fl = xs.sum_strided(d[:m], outer, length, inner, out64=True, out32=True, flags=True)
        v64 = o64.cpu().numpy().view(np.uint64)
        v32 = o32.cpu().numpy().view(np.uint32)
        f = fl.cpu().numpy().view(np.uint32)
        a3 = b[:m].reshape(outer, length, inner)
        for k in range(outer * inner):
            o, i = divmod(k, inner)
            r, _ = ref(fmt, np.ascontiguousarray(a3[o, :, i]))
            if (int(v64[k]), int(v32[k]), int(f[k])) != (r.bits, r.bits_f32, r.flags & 0xDF):
                return f"{fmt} strided {outer}x{length}x{inner} fibre {k}"
        return None
    if api == 6:                                          # checkpoint / resume mid-way
        c = int(rng.integers(0, n + 1))
        a = xs.Accumulator().add(d[:c])
        res, canon = xs.Accumulator().load_state(a.save_state()).add(d[c:]).exact()
        r, limbs = ref(fmt, b)
        return None if same(res, canon, r, limbs) else f"{fmt} n={n} checkpoint at {c}"
    if api == 0:
        res, canon = xs.exact_sum(d)
        r, limbs = ref(fmt, b)
        return None if same(res, canon, r, limbs) else f"{fmt} n={n} off={off} fused"
    if api == 1:
        cuts = np.sort(rng.integers(0, n + 1, size=int(rng.integers(1, 5))))
        acc = xs.Accumulator()
        prev = 0
        for c in list(cuts) + [n]:
            acc.add(d[prev:c])
            prev = c
        res, canon = acc.exact()
        r, limbs = ref(fmt, b)
        return None if same(res, canon, r, limbs) else f"{fmt} n={n} off={off} chunked {cuts}"
    if api == 2:
        host = d.cpu().pin_memory()
        res, canon = xs.Accumulator().add_host(host, stage_bytes=2 << 20).exact()
        r, limbs = ref(fmt, b)
        return None if same(res, canon, r, limbs) else f"{fmt} n={n} host"
    if api == 3:
        p = int(rng.integers(1, 6))
        cuts = [n * i // p for i in range(p + 1)]
        states = torch.cat([xs.Accumulator().add(d[cuts[i]:cuts[i + 1]]).state for i in range(p)])
        m = xs.Accumulator()
        if rng.random() < 0.5:
            m.merge(states)
        else:
            imgs, offs, o = [], [], 0
            for i in range(p):
                a = xs.Accumulator()
                a.merge(states[i * 384:(i + 1) * 384].clone())
                img, nb = a.to_sparse()
                imgs.append(img.cpu().numpy())
                offs.append(o)
                o += nb
            m.merge_sparse(torch.from_numpy(np.concatenate(imgs)).cuda(),
                           torch.tensor(offs, dtype=torch.int64, device="cuda"))
        res, canon = m.exact()
        r, limbs = ref(fmt, b)
        return None if same(res, canon, r, limbs) else f"{fmt} n={n} merge p={p}"
    # segments
    if n == 0:
        return None
    if api == 4:
        L = int(rng.integers(1, min(n, 9000) + 1))
        nseg = n // L
        if nseg == 0:
            return None
        bounds = [(s * L, (s + 1) * L) for s in range(nseg)]
        want_canon = bool(rng.integers(0, 2))         # values-only calls take other kernels (K11s, K9q)
        vals, canon, flags = xs.sum_segments(d[:nseg * L], L, canon=want_canon, flags=True)
    else:
        nseg = int(rng.integers(1, 40))
        cuts = np.sort(rng.integers(0, n + 1, size=nseg - 1))
        offs = np.concatenate([[0], cuts, [n]]).astype(np.int64)
        bounds = list(zip(offs[:-1], offs[1:]))
        vals, canon, flags = xs.sum_segments_csr(d, torch.from_numpy(offs).cuda(), canon=True, flags=True)
    v = vals.cpu().numpy()
    cn = canon.cpu().numpy().view(np.uint64) if canon is not None else None
    fl = flags.cpu().numpy().view(np.uint32)
    for s, (a, e) in enumerate(bounds):
        r, limbs = ref(fmt, b[a:e])
        want = r.bits if fmt == "f64" else r.bits_f32
        got = int(v[s:s + 1].view(np.uint64 if fmt == "f64" else np.uint32)[0])
        if got != want or fl[s] != r.flags or (cn is not None and not (cn[s] == limbs).all()):
            return f"{fmt} n={n} segments api={api} seg {s} [{a},{e})"
    return None


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
    base = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    xs.build()
    t0 = time.time()
    cases = fails = 0
    while time.time() - t0 < secs:
        seed = base + cases
        msg = one_case(seed)
        cases += 1
        if msg:
            fails += 1
            print(f"FAIL seed={seed}: {msg}", flush=True)
    print(f"fuzz: {cases} cases, {fails} failures in {time.time() - t0:.0f} s")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
