"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container, where /root/reference exists:
    python tests/golden/make_golden.py
It imports the reference package read-only (PYTHONPATH=/root/reference/pkg/src)
and records its outputs; the fixtures are committed so the tests never need
/root/reference at run time (it does not exist on the GPU box).

Fixtures:
  synthetic.json   SyntheticApp.compare values (apps.py:201-208) as exact hex doubles
  scheduler.json   iter_leaves (scheduler.py:78-86), pair_count, PairLedger.pair_id,
                   leaf_pair_total closed forms (test_scheduler.py:76-80)
  cv.json          CompositionVectorApp parse payloads + compare/postprocess matrices
                   for the reference tests' corpora (test_apps.py:47-53, test_engine.py:34-43,
                   test_acceptance.py:273-321)
  slotcache.json   a 4000-op randomized CacheTier trace (the test_slotcache.py:189-248
                   process) with every outcome and the final stats
  perfmodel.json   perfmodel t_gpu / t_min / efficiency values
"""

from __future__ import annotations

import json
import os
import random
import struct
import sys
import tempfile

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    from allpairs import perfmodel
    from allpairs.apps import CompositionVectorApp, ItemData, Stage, SyntheticApp
    from allpairs.rng import mix64
    from allpairs.scheduler import PairLedger, iter_leaves, leaf_pair_total, root_region
    from allpairs.slotcache import CacheTier, Hit, Miss, MustWait
    from allpairs.errors import NoEvictableSlot

    def dump(name, obj):
        with open(os.path.join(HERE, name), "w") as fh:
            json.dump(obj, fh, indent=None, separators=(",", ":"), sort_keys=True)
            fh.write("\n")

    # -- synthetic -------------------------------------------------------------
    cases = []
    for seed in (0, 1, 5, 2 ** 63 + 7, 0xFFFFFFFFFFFFFFFF):
        n = 24
        app = SyntheticApp(n=n, seed=seed)
        pre = app.preprocess(0, app.parse(0, ItemData(Stage.RAW_FILE, app.fetch_raw(app.path_for_key(0)))))
        vals = []
        for i in range(n):
            for j in range(i + 1, n):
                (v,) = struct.unpack("<d", app.compare((i, pre), (j, pre)))
                vals.append(v.hex())
        cases.append({"seed": seed, "n": n, "values": vals})
    payload = SyntheticApp(n=4, seed=9, payload_bytes=128).fetch_raw("items/000002.bin").hex()
    dump("synthetic.json", {"cases": cases, "mix64": [[list(a), mix64(*a)] for a in
                                                       [(0,), (1, 2), (5, 0xC0403A3E, 3, 4), (2 ** 64 - 1, 7)]],
                            "payload_seed9_key2_128": payload})

    # -- scheduler -------------------------------------------------------------
    leaves = {}
    for n in list(range(2, 41)) + [64, 100]:
        for lb in (1, 3, 8, 16):
            leaves[f"{n}/{lb}"] = [list(l.as_tuple()) for l in iter_leaves(root_region(n), lb)]
    pid = {}
    for n in (2, 5, 13, 100, 4096):
        ledger = PairLedger(n)
        rng = random.Random(n)
        pts = [(0, 1), (0, n - 1), (n - 2, n - 1)]
        for _ in range(40):
            i = rng.randrange(n - 1)
            j = rng.randrange(i + 1, n)
            pts.append((i, j))
        pid[str(n)] = [[i, j, ledger.pair_id(i, j)] for i, j in pts]
    totals = {str(n): leaf_pair_total(n, 8) for n in (256, 512, 2500, 4096)}
    dump("scheduler.json", {"leaves": leaves, "pair_id": pid, "leaf_pair_total_8": totals,
                            "pair_count": {str(n): root_region(n).pair_count()
                                           for n in (4980, 2500, 512, 256, 4096, 16384)}})

    # -- composition vectors -----------------------------------------------------
    five_docs = {"d0.txt": "ACGTACGTAAAC", "d1.txt": "TTTTGGGGCCCC", "d2.txt": "ACGTACGTAAAC",
                 "d3.txt": "GATTACAGATTACA", "d4.txt": "CCGGAATTCCGGTT"}

    def corpus(seed, count, length):
        out = {}
        for idx in range(count):
            state = mix64(seed, idx)
            chars = []
            for pos in range(length):
                state = mix64(state, pos)
                chars.append("ACGT"[state % 4])
            out[f"doc{idx:02d}.txt"] = "".join(chars)
        return out

    corpora = {
        "five_docs_k2": (five_docs, 2),
        "engine_seed0_k3": (corpus(0, 16, 120), 3),
        "acceptance_c04b05_k3": (corpus(0xC04B05, 16, 160), 3),
        "mixed_k4": ({"a.txt": "ACGTTGCAACGTTGCA" * 3, "b.txt": "acgt acgt\nacgt", "c.txt": "GGGGGGGGCCCC",
                      "d.txt": "ACGTTGCA" * 7 + "TTTT"}, 4),
    }
    cv = {}
    for name, (docs, k) in corpora.items():
        with tempfile.TemporaryDirectory() as tmp:
            for fn, text in docs.items():
                with open(os.path.join(tmp, fn), "w") as fh:
                    fh.write(text)
            app = CompositionVectorApp(tmp, k=k, threshold=0.5)
            parsed, pre = [], []
            for key in range(app.n):
                raw = ItemData(Stage.RAW_FILE, app.fetch_raw(app.path_for_key(key)))
                p = app.parse(key, raw)
                parsed.append(p.payload.hex())
                pre.append(app.preprocess(key, p))
            vals, matches = [], []
            for i in range(app.n):
                for j in range(i + 1, app.n):
                    raw = app.compare((i, pre[i]), (j, pre[j]))
                    res = app.postprocess((i, j), raw)
                    vals.append(res.value.hex())
                    matches.append(res.match)
            cv[name] = {"k": k, "texts": [docs[fn] for fn in sorted(docs)], "parsed": parsed,
                        "preprocessed": [x.payload.hex() for x in pre], "values": vals, "match": matches}
    dump("cv.json", cv)

    # -- slot cache trace --------------------------------------------------------
    rng = random.Random(1234)
    tier = CacheTier("dev", 4, 64)
    item = ItemData(Stage.PREPROCESSED, b"x" * 8)
    leases: dict[int, list] = {}
    tickets: dict[int, object] = {}
    ops = []
    for _ in range(4000):
        op = rng.random()
        key = rng.randrange(12)
        if op < 0.45:
            try:
                res = tier.acquire(key)
            except NoEvictableSlot:
                ops.append(["acquire", key, "noslot", -1])
                continue
            if isinstance(res, Hit):
                leases.setdefault(key, []).append(res.lease)
                ops.append(["acquire", key, "hit", res.lease.slot.index])
            elif isinstance(res, MustWait):
                ops.append(["acquire", key, "wait", tier.index[key].index])
            else:
                assert isinstance(res, Miss)
                tickets[key] = res.ticket
                ops.append(["acquire", key, "miss", res.ticket.slot.index])
        elif op < 0.70 and tickets:
            key = rng.choice(sorted(tickets))
            ticket = tickets.pop(key)
            if rng.random() < 0.8:
                retain = rng.random() < 0.3
                lease = tier.publish(ticket, item, retain=retain)
                if lease is not None:
                    leases.setdefault(key, []).append(lease)
                ops.append(["publish", key, int(retain), ticket.slot.index])
            else:
                ops.append(["abort", key, 0, ticket.slot.index])
                tier.abort(ticket)
        elif leases:
            candidates = [k for k, ls in leases.items() if ls]
            if candidates:
                key = rng.choice(candidates)
                lease = leases[key].pop()
                ops.append(["release", key, 0, lease.slot.index])
                lease.release()
    dump("slotcache.json", {"capacity": 4, "ops": ops, "final": tier.snapshot_stats(),
                            "final_keys": [s.key for s in tier.slots]})

    # -- performance model ---------------------------------------------------------
    costs = perfmodel.StageCosts(t_parse=0.13, t_preprocess=0.0205, t_comparison=0.0011, t_postprocess=1e-5,
                                 mean_file_bytes=3.0e7, io_bandwidth=4e8)
    rep = perfmodel.report(4980, 6.7, costs, p=16, t_measured=900.0)
    dump("perfmodel.json", {"costs": {"t_parse": 0.13, "t_preprocess": 0.0205, "t_comparison": 0.0011,
                                      "t_postprocess": 1e-5, "mean_file_bytes": 3.0e7, "io_bandwidth": 4e8},
                            "n": 4980, "R": 6.7, "p": 16, "t_measured": 900.0, "report": rep.as_dict()})
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
