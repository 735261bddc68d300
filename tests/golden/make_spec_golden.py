"""Writes tests/golden/spec_golden.json: every worked example of the
reference's SPEC.md that touches the GNS hot path or the goodput scorer.

The reference ships no code, fixtures or tests; its only
known-answer vectors are the [TRIVIAL]/[DERIVED] examples in SPEC.md.  This
script transcribes them (with the SPEC.md line each comes from) so the oracle
and the product are pinned to the same numbers.  Re-run:
    python tests/golden/make_spec_golden.py
"""
import json
import os

G = {
    "record_micro_batch": [
        {"src": "SPEC.md:171", "record": [4.0], "expect_s": [4.0], "expect_M": 1},
        {"src": "SPEC.md:172", "record": [1.5, 0.25, 7.0], "expect_s": [1.5, 0.25, 7.0], "expect_M": 3},
        {"src": "SPEC.md:173", "record": [-1.0], "expect_error": "ValidationError"},
    ],
    "finalize_step": [
        {"src": "SPEC.md:181", "dp_size": 1, "global_batch": 2,
         "micro_gradients": [[3.0, 0.0], [1.0, 0.0]],
         "expect": {"sbar": 5.0, "mean_grad_sq": 4.0, "signal": 3.0, "noise": 2.0, "noise_raw": 2.0}},
        {"src": "SPEC.md:182", "dp_size": 1, "global_batch": 4,
         "micro_gradients": [[0.5, -2.0, 1.0], [0.5, -2.0, 1.0], [0.5, -2.0, 1.0], [0.5, -2.0, 1.0]],
         "expect": {"mean_grad_sq": 5.25, "signal": 5.25, "noise": 0.0}},
        {"src": "SPEC.md:179", "dp_size": 1, "global_batch": 1,
         "micro_gradients": [[3.0, 0.0]], "expect_error": "ValidationError"},
    ],
    "update_ema": [
        {"src": "SPEC.md:191-192",
         "steps": [{"signal": 3.0, "noise": 2.0, "tokens": 4096},
                   {"signal": 5.0, "noise": 2.0, "tokens": 4096}],
         "expect_after": [{"ema_signal": 3.0, "ema_noise": 2.0},
                          {"ema_signal": 3.1, "ema_noise": 2.0}]},
        {"src": "SPEC.md:193 (phase switch)", "phase_boundary_tokens": 8000000,
         "steps": [{"signal": 1.0, "noise": 1.0, "tokens": 8000000},
                   {"signal": 2.0, "noise": 1.0, "tokens": 1}],
         "expect_alpha_second": 0.99},
    ],
    "gns": [
        {"src": "SPEC.md:201", "ema_signal": 3.0, "ema_noise": 2.0, "calibration": 2.0, "expect": 4.0 / 3.0},
        {"src": "SPEC.md:202", "ema_signal": 3.0, "ema_noise": 0.0, "calibration": 2.0, "expect": 0.0},
        {"src": "SPEC.md:203", "ema_signal": 0.0, "ema_noise": 2.0, "calibration": 2.0, "expect": None},
    ],
    "stat_eff": [
        {"src": "SPEC.md:259", "B_g": 1.0, "phi": 37.5, "expect": 1.0},
        {"src": "SPEC.md:260", "B_g": 64.0, "phi": 0.0, "expect": 1.0 / 64.0},
        {"src": "SPEC.md:261", "B_g": 100.0, "phi": 100.0, "expect": 0.505},
    ],
    "goodput": [
        {"src": "SPEC.md:269", "T": 500.0, "se": 0.5, "expect": 250.0},
    ],
    "goodput_lr": [
        {"src": "SPEC.md:281", "T": 500.0, "B_g": 64.0, "phi": 64.0, "ref": 16.0, "expect": 507.8125},
        {"src": "SPEC.md:279", "T": 300.0, "B_g": 16.0, "phi": 9.0, "ref": 16.0, "expect": 300.0 * 10.0 / 25.0},
    ],
    "lr_rescale": [
        {"src": "SPEC.md:289", "eta": 2e-4, "b_old": 16.0, "b_new": 64.0, "expect": 4e-4},
    ],
    "optimal_batch_continuous": [
        {"src": "SPEC.md:299", "b_hw": 64.0, "b_crit": 256.0, "expect": 128.0},
    ],
    "cbs_target": [
        {"src": "SPEC.md:309", "phi": 48.0, "cands": [16, 32, 64], "expect": 64},
        {"src": "SPEC.md:310", "phi": 0.0, "cands": [16, 32, 64], "expect": 16},
    ],
    "synth_profile": [
        {"src": "SPEC.md:80", "t_max": 1000.0, "b_hw": 64.0, "B_g": 64, "expect_T": 500.0},
        {"src": "SPEC.md:82", "p": 4, "ga": 1, "expect_bubble": 0.25},
        {"src": "SPEC.md:82", "p": 4, "ga": 16, "expect_bubble": 16.0 / 19.0},
    ],
    # decide: current score 100 at (S, B_g=16); scores are engineered with
    # phi = 0, ref = 16 so goodput_lr = T / sqrt(B_g * ref).
    "decide": [
        {"src": "SPEC.md:372", "same_strategy": True, "cand_score": 109.0, "elapsed": 1000.0,
         "useful": 1000.0, "reconfig_cost": 50.0, "expect": "NoOp"},
        {"src": "SPEC.md:373", "same_strategy": True, "cand_score": 115.0, "elapsed": 1000.0,
         "useful": 1000.0, "reconfig_cost": 50.0, "expect": "ScaleBS"},
        {"src": "SPEC.md:374", "same_strategy": False, "cand_score": 130.0, "elapsed": 1000.0,
         "useful": 1000.0, "reconfig_cost": 50.0, "expect": "Reconfigure",
         "expect_winner_score": 130.0 * 1000.0 / 1050.0},
        {"src": "SPEC.md:375", "same_strategy": False, "cand_score": 130.0, "elapsed": 30.0,
         "useful": 30.0, "reconfig_cost": 50.0, "expect": "NoOp",
         "expect_winner_score_max": 100.0},
    ],
}

if __name__ == "__main__":
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "spec_golden.json")
    with open(path, "w") as f:
        json.dump(G, f, indent=1, sort_keys=True)
    print("wrote", path)
