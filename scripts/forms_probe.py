"""Every kernel form on one small workload, checked against the oracle:
the three K2 forms (split chains, register-direct, smem-staged), both draw
plans, aggregated and Philox draws.  A quick GPU check after kernel edits:

    python scripts/forms_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))

import numpy as np
import torch

import oracle
import paper_1903_00227_b200 as wrs

P = oracle.port()
w = P.generate_powerlaw(300_000, 0.7, 5)
ref_b, ref_wn = P.psa_build(w, wrs.default_jobs(w.size))
for mode, env in (("split", {"WRS_B200_K2_SPLIT_MAX": "100000"}),
                  ("direct", {"WRS_B200_K2_SPLIT_MAX": "0"}),
                  ("staged", {"WRS_B200_K2_SPLIT_MAX": "0", "WRS_B200_K2_DIRECT_MAX": "0"})):
    os.environ.update(env)
    S = wrs.Sampler.build(wrs.Weights.from_array(w), "psa", 1)
    assert S.buckets().tobytes() == ref_b.tobytes(), mode
    print("table ok", mode, flush=True)
for plan in ("direct", "region"):
    os.environ["WRS_B200_PLAN"] = plan
    k = 200_003
    out = S.draw(7, k, 3)
    assert np.array_equal(out, P.sample_many(ref_b, ref_wn, 7, k, 3)), plan
    items, counts = S.draw_counts(7, k, 3)
    assert int(counts.sum()) == k
    d = torch.empty(k, dtype=torch.int32, device="cuda")
    S.draw_philox_device(9, k, d)
    torch.cuda.synchronize()
    print("draws ok", plan, flush=True)
print("forms probe ok")
