"""Wire/disk formats around phi: profile CSV
(acceptance #10 round trip) and the decision audit
log."""
import os

import pytest

from paper_2604_26687_b200 import gns as G
from paper_2604_26687_b200._lib import ValidationError

HDR = "d,t,p,global_batch,micro_batch,samples_per_sec,peak_mem_bytes,feasible\n"


def test_spec_row_maps_to_entry():
    # row 2,1,4,16,2,310.5,41e9,1
    ents, n = G.parse_profile_csv(HDR + "2,1,4,16,2,310.5,41e9,1\n")
    assert n == 8 and len(ents) == 1
    e = ents[0]
    assert (e.d, e.t, e.p, e.global_batch, e.micro_batch) == (2, 1, 4, 16, 2)
    assert e.samples_per_sec == 310.5 and e.peak_mem_bytes == 41e9 and e.feasible


def test_spec_validation_errors():
    with pytest.raises(ValidationError, match="line 2"):  # SPEC.md:71, 17 mod 4 != 0
        G.parse_profile_csv(HDR + "2,1,4,17,2,310.5,41e9,1\n")
    with pytest.raises(ValidationError, match="duplicate"):
        G.parse_profile_csv(HDR + "2,1,4,16,2,310.5,41e9,1\n2,1,4,16,2,300,41e9,1\n")
    with pytest.raises(ValidationError, match="line 3"):  # d*t*p differs from row 1
        G.parse_profile_csv(HDR + "2,1,4,16,2,310.5,41e9,1\n1,1,4,16,2,1,1,1\n")
    with pytest.raises(ValidationError, match="line 2"):  # malformed number
        G.parse_profile_csv(HDR + "2,1,4,16,2,31x,41e9,1\n")
    with pytest.raises(ValidationError, match="header"):
        G.parse_profile_csv("d,t,p\n")


def test_round_trip_is_bit_exact(tmp_path):
    costs = [(8, 1, 1, 4000.0, 256.0), (4, 2, 1, 3300.0, 96.0), (2, 2, 2, 2600.0, 40.0)]
    cands = G.synth_candidates(costs, [16, 32, 64, 128], [1, 2, 4], True)
    ents = [G.ProfileEntry(c.d, c.t, c.p, c.global_batch, c.micro_batch, c.throughput,
                           1e9 / 3.0 * c.micro_batch, True) for c in cands]
    ents.append(G.ProfileEntry(8, 1, 1, 2048, 8, 0.0, 9.9e10, False))
    text = G.profile_csv(ents)
    back, n = G.parse_profile_csv(text)
    assert n == 8
    key = lambda e: (e.d, e.t, e.p, e.global_batch, e.micro_batch)
    assert sorted(back, key=key) == sorted(ents, key=key)
    assert G.profile_csv(back) == text  # byte-identical re-serialisation
    path = os.path.join(tmp_path, "profile.csv")
    G.save_profile(path, ents)
    assert open(path).read() == text
    assert G.load_profile(path)[0] == back


def test_decision_audit_log():
    cands = G.synth_candidates([(8, 1, 1, 4000.0, 256.0), (4, 2, 1, 3300.0, 96.0)],
                               [16, 32, 64], [1, 2], True)
    cur = cands[0]
    cmd = G.decide(cands, 64.0, cur, 1000.0, 900.0, reconfig_cost=40.0)
    rows = [G.DecisionRow(25, 12.5, 64.0, cur, cands[max(cmd.winner_index, 0)], cmd),
            G.DecisionRow(50, 25.0, None, cur, cur, G.decide(cands, None, cur, 1.0, 1.0))]
    text = G.decision_audit_csv(rows)
    lines = text.splitlines()
    assert lines[0] == ("step,time_s,phi,current_cfg,winner_cfg,current_score,winner_score,"
                        "penalized,command")
    f = lines[1].split(",")
    assert (f[0], f[1], f[2]) == ("25", "12.5", "64")
    assert f[3] == f"d{cur.d}t{cur.t}p{cur.p}_g{cur.global_batch}_m{cur.micro_batch}"
    assert f[8] == cmd.name
    assert float(f[5]) == cmd.current_score
    assert lines[2].split(",")[2] == "nan" and lines[2].endswith("NoOp")
