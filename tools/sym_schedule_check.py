"""Host model of the symmetric sweep's tile-visit protocol (csrc/sym_path.cu).

Restates SymWave (tiles, rotated steps, ranks) and the list agent's
load/release state machine, then checks that
  * every rectangle tile's visit ranks within the kernel form 0..K-1, and
  * the agents cannot deadlock: a greedy scheduler of the monotone version
    counters runs every agent to completion (with monotone waits, any fair
    schedule then completes too).
Used by tests/test_sym_schedule.py; `python tools/sym_schedule_check.py N...`.
"""
from __future__ import annotations

import sys
from collections import defaultdict

BM, BN = 128, 256


def visit_sequences(n: int, sms: int = 148, spread: int = 2):
    nrb, T = (n + BM - 1) // BM, (n + BN - 1) // BN
    G = min(nrb, sms)
    if G < nrb:
        G &= ~1
    waves = (nrb + G - 1) // G
    seqs = []
    for c in range(G):
        seq = []
        for w in range(waves):
            Gw = min(G, nrb - w * G)
            if c >= Gw:
                continue
            t_hi = (w * G + Gw - 1) // 2
            L = T - t_hi - 1 if T > t_hi + 1 else 0
            rot = spread * Gw <= L
            for s in range(L):
                qq = (s + spread * c) % L if rot else s
                if rot:
                    c1 = min(qq // spread, Gw - 1)
                    rk = c1 - c if c <= c1 else c1 + 1 + (Gw - 1 - c)
                else:
                    rk = c
                seq.append((t_hi + 1 + qq, G * w + rk, w))
        seqs.append(seq)
    return seqs


def check(n: int, sms: int = 148, spread: int = 2) -> str:
    seqs = visit_sequences(n, sms, spread)
    per = defaultdict(list)
    for seq in seqs:
        for t, v, _ in seq:
            per[t].append(v)
    for t, vs in per.items():
        if sorted(vs) != list(range(len(vs))):
            return f"bad ranks on tile {t}"
    # agent state machine (csrc/sym_path.cu): load visit `nload` once the
    # tile's version equals its rank and a buffer is free (nload < nrel + 2);
    # release visit `nrel` once loaded (merging is local progress).  The
    # waves of one CTA run one after another.
    version = defaultdict(int)
    G = len(seqs)
    nload, nrel, done = [0] * G, [0] * G, [False] * G
    progress = True
    while progress:
        progress = False
        for c in range(G):
            seq = seqs[c]
            if done[c]:
                continue
            if nrel[c] == len(seq):
                done[c] = progress = True
                continue
            if nload[c] < len(seq) and nload[c] < nrel[c] + 2:
                t, v, w = seq[nload[c]]
                same_wave = nload[c] == nrel[c] or seq[nrel[c]][2] == w
                if same_wave and version[t] == v:
                    nload[c] += 1
                    progress = True
            if nrel[c] < nload[c]:
                t, v, _ = seq[nrel[c]]
                version[t] = v + 1
                nrel[c] += 1
                progress = True
    if not all(done):
        stuck = [c for c in range(G) if not done[c]]
        return f"deadlock: {len(stuck)} agents stuck, e.g. CTA {stuck[0]} at visit {nload[stuck[0]]}"
    return "ok"


if __name__ == "__main__":
    for a in sys.argv[1:]:
        print(a, check(int(a)))
