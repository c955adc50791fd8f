"""Generates tests/golden/zipper_ref.json and numerics_ref.json from the REFERENCE itself
(proj/include compiled in place into oracle/_ref/libref.so by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures are committed; the GPU box never needs /root/reference.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def signatures(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        ul = int(rng.integers(0, 40))
        al = int(rng.integers(0, 40))
        u = bytes(rng.integers(32, 127, ul, dtype=np.uint8))
        a = bytes(rng.integers(32, 127, al, dtype=np.uint8))
        ts = int(rng.integers(-2**62, 2**62))
        out.append((u, a, ts))
    # hand-picked: survey goldens, empty strings, long path, extremes
    out += [(b"u1", b"a1", 0), (b"user_000042", b"ad_9", 1700000000000), (b"", b"x", -5),
            (b"alice", b"campaign-7/creative-13", 86400000), (b"", b"", 0),
            (b"u" * 200, b"a" * 300, 2**63 - 1), (b"", b"", -2**63)]
    return out


def main():
    ref = oracle.load_ref()
    sigs = signatures(200, 11)
    configs = [
        {"durations": [5400000, 86400000], "probs": [0.5, 0.5], "seed": 7},
        {"durations": [1, 2, 3, 4], "probs": [0.4, 0.3, 0.2, 0.1], "seed": 7},
        {"durations": [5400000, 86400000, 604800000], "probs": [1 / 3, 1 / 3, 1 / 3], "seed": 7},
        {"durations": [10, 20], "probs": [1.0, 0.0], "seed": 2024},
    ]
    cases = []
    for u, a, ts in sigs:
        buf = np.zeros(16 + len(u) + len(a), np.uint8)
        n = ref.ref_signature(u, len(u), a, len(a), ts, oracle.ptr(buf))
        h = {}
        wins = []
        for c in configs:
            dur = np.array(c["durations"], np.int64)
            pr = np.array(c["probs"], np.float64)
            w = oracle._I64(-1)
            rc = ref.ref_assign_window(u, len(u), a, len(a), ts, len(dur), oracle.ptr(dur),
                                       oracle.ptr(pr), c["seed"], oracle.ctypes.byref(w))
            assert rc == 0
            wins.append(int(w.value))
        h = ref.ref_stable_hash(oracle.ptr(buf), n, 7)
        cases.append({"user": u.hex(), "ad": a.hex(), "ts": ts, "sig": buf[:n].tobytes().hex(),
                      "xxh64_seed7": f"{h:016x}", "windows": wins})

    # label cases through zip_dataset (datasets.hpp:199)
    rng = np.random.default_rng(5)
    n, T, W = 64, 3, 3
    users = [f"u{int(x)}".encode() for x in rng.integers(0, 10**8, n)]
    ads = [f"a{int(x)}".encode() for x in rng.integers(0, 10**6, n)]
    ts = 1_700_000_000_000 + 37 * np.arange(n, dtype=np.int64)
    durations = np.array([5400000, 86400000, 604800000], np.int64)
    pres = (rng.random((n, T)) < 0.6).astype(np.uint8)
    delay = rng.integers(0, 8 * 86400000, (n, T))
    delay[0, 0] = 5400000  # closed boundary
    delay[1, 1] = 86400000
    delay[2, 2] = 604800001
    pres[0:3] = 1
    conv = ts[:, None] + delay
    rc, win, lab, msg = oracle.ref_zip_dataset(users, ads, ts, conv, pres, durations,
                                               [1 / 3, 1 / 3, 1 / 3], 7)
    assert rc == 0, msg
    zip_case = {"users": [u.decode() for u in users], "ads": [a.decode() for a in ads],
                "ts": ts.tolist(), "conv": conv.tolist(), "present": pres.tolist(),
                "durations": durations.tolist(), "probs": [1 / 3, 1 / 3, 1 / 3], "seed": 7,
                "window": win.tolist(), "labels": lab.tolist()}
    conv_bad = conv.copy()
    conv_bad[40, 2] = ts[40] - 1
    conv_bad[41, 0] = ts[41] - 5
    pres_bad = pres.copy()
    pres_bad[40, 2] = 1
    pres_bad[41, 0] = 1
    rc, _, _, msg = oracle.ref_zip_dataset(users, ads, ts, conv_bad, pres_bad, durations,
                                           [1 / 3, 1 / 3, 1 / 3], 7)
    assert rc == 2
    zip_err = {"conv": conv_bad.tolist(), "present": pres_bad.tolist(), "message": msg}

    with open(os.path.join(HERE, "zipper_ref.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py via oracle/_ref/libref.so",
                   "configs": configs, "signatures": cases, "zip": zip_case,
                   "zip_error": zip_err}, f, indent=0)

    # numerics (numerics.hpp:81-107)
    rng = np.random.default_rng(3)
    vecs = [[3.0, 4.0], [2.0, 2.0], [0.0, 0.0, 0.0], [1e6] * 7 + [-1e6]]
    vecs += [list(rng.uniform(-10, 10, int(rng.integers(1, 300)))) for _ in range(12)]
    num = []
    for v in vecs:
        row = {"x": v}
        for name in ("ref_rms_norm", "ref_swish_rn", "ref_swish_rn_hard"):
            rc, out = oracle.vec_op(ref, name, v)
            assert rc == 0
            row[name[4:]] = out.tolist()
        num.append(row)
    with open(os.path.join(HERE, "numerics_ref.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py via oracle/_ref/libref.so",
                   "eps": 1e-6, "cases": num}, f)
    print("wrote", len(cases), "signature cases,", len(num), "numerics cases")


if __name__ == "__main__":
    main()
