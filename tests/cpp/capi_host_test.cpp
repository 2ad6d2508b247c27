// C++ host test of the reference-facing API (include/appo_b200.hpp over the
// C ABI): known-answer V-trace (test_offpolicy.cpp:71-86), the reference
// exception taxonomy, and one batched inference + learner step.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "appo_b200.hpp"

#define REQUIRE(c)                                                     \
  do {                                                                 \
    if (!(c)) {                                                        \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                        \
    }                                                                  \
  } while (0)

int main() {
  using namespace appo_b200;
  Context ctx(0, 1);
  // known answer: v = [2, 1], pg_adv = [2, 1]
  std::vector<double> r{1.0, 1.0}, v{0.0, 0.0}, tl{-0.5, -0.7}, bl{-0.5, -0.7};
  std::vector<uint8_t> d{0, 0};
  auto out = ctx.vtrace(r, v, 0.0, tl, bl, d, VTraceConfig{1.0, 1.0, 1.0});
  REQUIRE(std::fabs(out.v[0] - 2.0) < 1e-6 && std::fabs(out.v[1] - 1.0) < 1e-6);
  REQUIRE(std::fabs(out.pg_adv[0] - 2.0) < 1e-6 && std::fabs(out.pg_adv[1] - 1.0) < 1e-6);
  REQUIRE(out.rho[0] == 1.0 && out.c[1] == 1.0);
  // error taxonomy: rho_bar < c_bar -> ConfigError; NaN -> NumericError; shape -> ContractError
  bool got = false;
  try { ctx.vtrace(r, v, 0.0, tl, bl, d, VTraceConfig{0.5, 1.0, 0.99}); } catch (const ConfigError&) { got = true; }
  REQUIRE(got);
  got = false;
  std::vector<double> rn{NAN, 1.0};
  try { ctx.vtrace(rn, v, 0.0, tl, bl, d, VTraceConfig{}); } catch (const NumericError&) { got = true; }
  REQUIRE(got);
  got = false;
  std::vector<double> r3{1.0, 1.0, 1.0};
  try { ctx.vtrace(r3, v, 0.0, tl, bl, d, VTraceConfig{}); } catch (const ContractError&) { got = true; }
  REQUIRE(got);

  // nstep_returns KAT (test_offpolicy.cpp:254-261)
  {
    std::vector<double> rw{1.0, 1.0, 1.0};
    std::vector<uint8_t> dn{0, 1, 0};
    auto ret = ctx.nstep_returns(rw, 10.0, dn, 0.5);
    REQUIRE(std::fabs(ret[2] - 6.0) < 1e-6 && std::fabs(ret[1] - 1.0) < 1e-6 &&
            std::fabs(ret[0] - 1.5) < 1e-6);
  }
  // heads: uniform entropies (test_policy.cpp:241-252), degenerate logits
  // (:195-203), reproducible sampling under a fixed seed over the full
  // factored space (:226-239), out-of-range action (:292-297)
  {
    ActionHeadsSpec h22{{2, 2}};
    auto [lp, ent] = ctx.log_prob_and_entropy(h22, std::vector<double>{0, 0, 0, 0}, {0, 1});
    REQUIRE(std::fabs(ent - 2.0 * std::log(2.0)) < 1e-6 && std::fabs(lp - 2.0 * std::log(0.5)) < 1e-6);
    ActionHeadsSpec h3{{3}};
    std::mt19937_64 rng(11);
    auto [a, lpa] = ctx.sample_action(h3, std::vector<double>{1e9, 0.0, 0.0}, rng);
    REQUIRE(a.size() == 1 && a[0] == 0 && std::fabs(lpa) < 1e-6);
    ActionHeadsSpec full{{3, 3, 2, 2, 2, 8, 21}};
    std::vector<double> lg(full.logits_dim());
    std::mt19937_64 lrng(5);
    for (auto& l : lg) l = std::uniform_real_distribution<double>(-1, 1)(lrng);
    std::mt19937_64 ra(99), rb(99);
    for (int i = 0; i < 5; ++i) {
      auto [a1, l1] = ctx.sample_action(full, lg, ra);
      auto [a2, l2] = ctx.sample_action(full, lg, rb);
      REQUIRE(a1 == a2 && l1 == l2 && a1.size() == 7);
      for (int j = 0; j < 7; ++j) REQUIRE(a1[j] >= 0 && a1[j] < full.sizes[j]);
    }
    bool thrown = false;
    try { ctx.log_prob_and_entropy(h3, std::vector<double>{0, 0, 0}, {3}); } catch (const ContractError&) { thrown = true; }
    REQUIRE(thrown);
  }
  // optimizer_step: zero gradient leaves theta, bumps version
  // (test_policy.cpp:382-390); norm 8 under clip 4 equals norm 4 unclipped
  // (:392-413); non-finite gradient throws NumericError, p untouched
  {
    PolicyParams p;
    p.theta.assign(1000, 0.0);
    // fp32-representable values: the device keeps theta in fp32
    for (size_t i = 0; i < p.theta.size(); ++i) p.theta[i] = static_cast<double>(i) / 1024.0;
    const auto before = p.theta;
    ctx.optimizer_step(p, std::vector<double>(1000, 0.0), AdamConfig{});
    REQUIRE(p.theta == before && p.version == 1 && p.adam.t == 1);
    PolicyParams pa = p, pb = p;
    std::vector<double> g(1000, 0.0), half(1000, 0.0);
    g[0] = 8.0; half[0] = 4.0;
    AdamConfig clip4, noclip;
    clip4.grad_clip = 4.0; noclip.grad_clip = 0.0;
    ctx.optimizer_step(pa, g, clip4);
    ctx.optimizer_step(pb, half, noclip);
    REQUIRE(pa.theta == pb.theta && pa.theta != p.theta);
    g[3] = NAN;
    PolicyParams pc = p;
    bool thrown = false;
    try { ctx.optimizer_step(pc, g, clip4); } catch (const NumericError&) { thrown = true; }
    REQUIRE(thrown && pc.theta == p.theta && pc.version == p.version);
  }

  // model: one inference batch and one learner step through the C ABI
  appo_model_desc desc{3, 72, 128, 6, 8, {0, 0, 0}};
  Context m(0, 7, &desc);
  const int B = 16;
  const size_t od = 3 * 72 * 128;
  DeviceBuffer<uint8_t> obs(B * od);
  DeviceBuffer<float> h(B * 512), hout(B * 512), lp(B), val(B);
  DeviceBuffer<int32_t> act(B);
  std::vector<uint8_t> hobs(B * od);
  for (size_t i = 0; i < hobs.size(); ++i) hobs[i] = static_cast<uint8_t>((i * 2654435761u) >> 24);
  obs.upload(hobs.data());
  cudaMemset(h.get(), 0, B * 512 * 4);
  const int64_t ver = m.policy_forward(B, obs.get(), h.get(), 0, act.get(), lp.get(), hout.get(), val.get());
  m.sync();
  REQUIRE(ver == 0);
  std::vector<int32_t> ha(B);
  act.download(ha.data());
  for (int a : ha) REQUIRE(a >= 0 && a < 6);
  std::vector<float> theta;
  REQUIRE(m.fetch(theta) == 0 && theta.size() == 2872551);
  // checkpoint round trip into a differently seeded context
  const std::string ck = "/tmp/capi_host_test.ckpt";
  m.save_checkpoint(ck);
  Context m2(0, 77, &desc);
  std::vector<float> theta2;
  m2.load_checkpoint(ck);
  REQUIRE(m2.fetch(theta2) == 0 && theta2 == theta);
  std::remove(ck.c_str());

  // PBT over two learners: policy 0 scores higher, policy 1 takes its weights
  appo_pbt_config pc{};
  pc.pbt_period = 100; pc.mutate_fraction = 0.0; pc.mutation_rate = 0.15;
  pc.mutation_factor = 1.2; pc.replace_fraction = 0.5; pc.window = 10;
  Context l0(0, 5, &desc), l1(0, 6, &desc);
  PbtController pbt(pc, {&l0, &l1}, appo_pbt_controller_seed(1));
  pbt.record(0, 1.0);
  pbt.record(1, 0.0);
  REQUIRE(pbt.tick(50).empty());
  const auto ev = pbt.tick(100);
  REQUIRE(ev.size() == 1 && ev[0].event == 1 && ev[0].agent == 1);
  std::vector<float> p0, p1;
  l0.fetch(p0);
  l1.fetch(p1);
  REQUIRE(p0 == p1);

  // device ready queue: ids pushed on the device come back in FIFO order
  SlotQueue q(0, 8);
  DeviceBuffer<int32_t> ids(3), popped(3);
  const int32_t h_ids[3] = {5, 2, 7};
  ids.upload(h_ids);
  q.push(m, ids.get(), 3);
  q.pop(m, popped.get(), 3);
  m.sync();
  int32_t h_got[3];
  popped.download(h_got);
  REQUIRE(h_got[0] == 5 && h_got[1] == 2 && h_got[2] == 7);
  std::printf("capi_host_test ok\n");
  return 0;
}
