// dropin_main.cpp — drop-in check of the C++ boundary.
//
// Written against the reference's public API only (proj/include/coadapt/
// gns.hpp, goodput.hpp, strategy.hpp, io.hpp, errors.hpp).  tests/test_dropin.py
// compiles it twice — against include/coadapt/ of this repo and, when
// /root/reference is present, against the reference's own headers — and
// links both builds to libcoadapt_b200.so.  Linking proves every declared
// symbol is implemented with the reference's signatures; running checks the
// SPEC.md worked examples.  `--gpu` additionally exercises the span overload
// of finalize_step, which reduces on the device.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "coadapt/errors.hpp"
#include "coadapt/gns.hpp"
#include "coadapt/goodput.hpp"
#include "coadapt/io.hpp"
#include "coadapt/strategy.hpp"

static int failures = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    if (!(cond)) {                                                      \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #cond);        \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  using namespace coadapt;

  // record_micro_batch
  StepAccumulator acc(1, 2);
  acc.record_micro_batch(9.0);
  acc.record_micro_batch(1.0);
  CHECK(acc.sample_count() == 2 && acc.micro_count() == 2);
  bool threw = false;
  try {
    acc.record_micro_batch(-1.0);
  } catch (const ValidationError&) {
    threw = true;
  }
  CHECK(threw);

  // finalize_step scalar overload, SPEC.md:181 (exact)
  StepStats st = finalize_step(acc, 4.0);
  CHECK(st.signal == 3.0 && st.noise == 2.0 && st.noise_raw == 2.0);
  threw = false;
  try {
    StepAccumulator one(1, 1);
    one.record_micro_batch(1.0);
    finalize_step(one, 1.0);
  } catch (const ValidationError&) {
    threw = true;
  }
  CHECK(threw);

  // update_ema + gns
  GnsState gs;
  update_ema(gs, st, 4096);
  CHECK(gs.ema_signal == 3.0 && gs.ema_noise == 2.0 && gs.initialized);
  StepStats st2{5.0, 2.0, 2.0, 0.0};
  update_ema(gs, st2, 4096);
  CHECK(std::fabs(gs.ema_signal - 3.1) < 1e-15);
  GnsState g2;
  g2.ema_signal = 3.0;
  g2.ema_noise = 2.0;
  CHECK(gns(g2).has_value() && std::fabs(*gns(g2) - 4.0 / 3.0) < 1e-15);
  g2.ema_signal = 0.0;
  CHECK(!gns(g2).has_value());

  // goodput
  CHECK(std::fabs(stat_eff(100.0, 100.0) - 0.505) < 1e-15);
  CHECK(goodput(500.0, 0.5) == 250.0);
  CHECK(goodput_lr(500.0, 64.0, 64.0, 16.0) == 507.8125);
  CHECK(std::fabs(lr_rescale(2e-4, 16, 64) - 4e-4) < 1e-18);
  CHECK(optimal_batch_continuous(64, 256) == 128.0);
  const std::vector<std::int64_t> cands{16, 32, 64};
  CHECK(cbs_target(48.0, cands) == 64);
  CHECK(cbs_target(0.0, cands) == 16);
  EfficiencyContext ctx;
  CHECK(std::fabs(ctx.lr_at(64.0) - 4e-4) < 1e-18);

  // strategy
  ParallelStrategy s{2, 1, 4};
  CHECK(s.label() == "d2t1p4" && s.gpus() == 8);
  ConfigTuple c{s, 16, 2};
  CHECK(c.divisible() && c.grad_accum() == 4 && c.label() == "d2t1p4_g16_m2");
  CHECK(parse_strategy_label("2,1,4") == s && parse_strategy_label("d2t1p4") == s);
  threw = false;
  try {
    validate_config(ConfigTuple{s, 17, 2}, 8);
  } catch (const ValidationError&) {
    threw = true;
  }
  CHECK(threw);

  // io, io.hpp:13-25
  CHECK(format_double(0.1) == "0.1" && format_int(-42) == "-42");
  CHECK(parse_double("1e-3", "x") == 1e-3 && parse_int("17", "x") == 17);
  threw = false;
  try {
    parse_double("1.5x", "profile.csv line 7");
  } catch (const ParseError&) {
    threw = true;
  }
  CHECK(threw);
  CHECK(split_csv_line("a,b,,c").size() == 4);

  // trace CSV, gns.hpp:82-94
  std::vector<GnsTraceRow> rows(1);
  rows[0].step = 1;
  rows[0].tokens = 4096;
  rows[0].signal_raw = 3.0;
  rows[0].noise_raw = 2.0;
  rows[0].ema_signal = 3.0;
  rows[0].ema_noise = 2.0;
  rows[0].phi = std::nan("");
  CHECK(gns_trace_csv(rows) ==
        "step,tokens,signal_raw,noise_raw,ema_signal,ema_noise,phi\n"
        "1,4096,3,2,3,2,nan\n");

  // simulate_micro_gradients
  const std::vector<double> G{1.0, -2.0}, Z{0.0, 0.0};
  const auto draws = simulate_micro_gradients(G, Z, 4, 3, 7);
  CHECK(draws.size() == 3 && draws[2][1] == -2.0);

  if (gpu) {
    // span overload: ||mean||^2 reduced on the B200
    const std::vector<double> mean{2.0, 0.0};
    const StepStats sg = finalize_step(acc, mean);
    CHECK(sg.signal == 3.0 && sg.noise == 2.0 && sg.mean_grad_sq == 4.0);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
