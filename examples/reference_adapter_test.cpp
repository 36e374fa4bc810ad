// The reference's own layer code (ref:proj/core/src/{ops,layers}.cpp, compiled in place into
// oracle/_ref) against the B200 path reached through the reference-typed adapter
// (examples/reference_adapter.hpp -> include/revprop_b200.hpp -> librevprop_b200.so), on the
// same inputs. Built on CPU by tests/test_capi.py (needs /root/reference), run on the B200 by
// tests/test_gpu_adapter.py. Exit status 0 iff every check passes; one line per check.
//
// Weights are rounded to bf16 values on the host first, so both sides multiply the same
// numbers (the B200 GEMMs take bf16 operands); the remaining difference is the B200's bf16
// activation operands vs the reference's fp32, held to the stated tolerance.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "reference_adapter.hpp"
#include "revprop/ops.hpp"
#include "revprop/rng.hpp"

using namespace revprop;
namespace A = revprop::b200_adapter;
namespace B = revprop::b200;

static int g_fail = 0;

static void report(const char* what, double err, double tol) {
  const bool ok = err <= tol;
  std::printf("%-44s %.3e (tol %.1e) %s\n", what, err, tol, ok ? "ok" : "FAIL");
  if (!ok) ++g_fail;
}
static void report_bool(const char* what, bool ok) {
  std::printf("%-44s %s\n", what, ok ? "ok" : "FAIL");
  if (!ok) ++g_fail;
}

static Tensor bf16_round(Tensor t) {
  for (std::size_t i = 0; i < t.numel(); ++i) {
    float f = static_cast<float>(t.get(i));
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
    std::memcpy(&f, &u, 4);
    t.set(i, f);
  }
  return t;
}

static AttentionParams attn_params(std::size_t d, std::size_t heads, std::optional<std::size_t> w,
                                   Rng& rng) {
  AttentionParams p;
  p.w_qkv = bf16_round(ops::trunc_normal({d, 3 * d}, Dtype::f32, rng, 0.02));
  p.w_out = bf16_round(ops::trunc_normal({d, d}, Dtype::f32, rng, 0.02));
  p.ln_gamma = ops::randn({d}, Dtype::f32, rng, 0.1);
  for (std::size_t i = 0; i < d; ++i) p.ln_gamma.set(i, 1.0 + p.ln_gamma.get(i));
  p.ln_beta = ops::randn({d}, Dtype::f32, rng, 0.1);
  p.heads = heads;
  p.window = w;
  return p;
}

static MlpParams mlp_params(std::size_t d, std::size_t h, Rng& rng) {
  MlpParams p;
  p.w1 = bf16_round(ops::trunc_normal({d, h}, Dtype::f32, rng, 0.02));
  p.b1 = ops::randn({h}, Dtype::f32, rng, 0.02);
  p.w2 = bf16_round(ops::trunc_normal({h, d}, Dtype::f32, rng, 0.02));
  p.b2 = ops::randn({d}, Dtype::f32, rng, 0.02);
  p.ln_gamma = ops::randn({d}, Dtype::f32, rng, 0.1);
  for (std::size_t i = 0; i < d; ++i) p.ln_gamma.set(i, 1.0 + p.ln_gamma.get(i));
  p.ln_beta = ops::randn({d}, Dtype::f32, rng, 0.1);
  return p;
}

static double rel(const Tensor& a, const Tensor& b) { return ops::max_rel_diff(a, b); }

static void check_attention(const char* name, std::size_t Bn, std::size_t N, std::size_t d,
                            std::size_t heads, std::optional<std::size_t> window) {
  Rng rng(7, 1);
  const AttentionParams p = attn_params(d, heads, window, rng);
  const Tensor x = ops::randn({Bn, N, d}, Dtype::f32, rng);
  const Tensor dy = ops::randn({Bn, N, d}, Dtype::f32, rng);
  const AttentionForward rf = attention_forward(x, p);           // the reference, CPU
  const AttentionVjp rv = attention_vjp(rf.cache, p, dy);
  const A::AttentionForwardB200 gf = A::attention_forward(x, p);  // the B200, same types
  const AttentionVjp gv = A::attention_vjp(gf.cache, p, dy);
  const std::string n(name);
  report((n + " y").c_str(), rel(gf.y, rf.y), 2e-2);
  report((n + " d_x").c_str(), rel(gv.d_x, rv.d_x), 2e-2);
  report((n + " d_w_qkv").c_str(), rel(gv.d_params.d_w_qkv, rv.d_params.d_w_qkv), 2e-2);
  report((n + " d_w_out").c_str(), rel(gv.d_params.d_w_out, rv.d_params.d_w_out), 2e-2);
  report((n + " d_ln_gamma").c_str(), rel(gv.d_params.d_ln_gamma, rv.d_params.d_ln_gamma), 5e-2);
  report((n + " d_ln_beta").c_str(), rel(gv.d_params.d_ln_beta, rv.d_params.d_ln_beta), 5e-2);
}

static void check_mlp() {
  Rng rng(8, 1);
  const MlpParams p = mlp_params(192, 768, rng);
  const Tensor x = ops::randn({2, 197, 192}, Dtype::f32, rng);
  const Tensor dy = ops::randn({2, 197, 192}, Dtype::f32, rng);
  const MlpForward rf = mlp_forward(x, p);
  const MlpVjp rv = mlp_vjp(rf.cache, p, dy);
  const A::MlpForwardB200 gf = A::mlp_forward(x, p);
  const MlpVjp gv = A::mlp_vjp(gf.cache, p, dy);
  report("mlp y", rel(gf.y, rf.y), 2e-2);
  report("mlp d_x", rel(gv.d_x, rv.d_x), 2e-2);
  report("mlp d_w1", rel(gv.d_params.d_w1, rv.d_params.d_w1), 2e-2);
  report("mlp d_b1", rel(gv.d_params.d_b1, rv.d_params.d_b1), 5e-2);
  report("mlp d_w2", rel(gv.d_params.d_w2, rv.d_params.d_w2), 2e-2);
  report("mlp d_b2", rel(gv.d_params.d_b2, rv.d_params.d_b2), 1e-5);
  report("mlp d_ln_gamma", rel(gv.d_params.d_ln_gamma, rv.d_params.d_ln_gamma), 5e-2);
  report("mlp d_ln_beta", rel(gv.d_params.d_ln_beta, rv.d_params.d_ln_beta), 5e-2);
}

// SPEC.md:213-239 restated on the reference's own layer functions (the reference specifies
// revcore but ships no code for it)
static A::Coupled ref_rev_forward(const A::RevBlock& b, const A::Coupled& in) {
  Tensor o2 = ops::add(in.i2, attention_forward(in.i1, b.f).y);
  Tensor o1 = ops::add(in.i1, mlp_forward(o2, b.g).y);
  return {o1, o2};
}

static void check_revcore() {
  Rng rng(9, 1);
  A::RevBlock blk{attn_params(192, 3, std::nullopt, rng), mlp_params(192, 768, rng), 1};
  const A::Coupled in{ops::randn({2, 197, 192}, Dtype::f32, rng),
                      ops::randn({2, 197, 192}, Dtype::f32, rng)};
  const A::Coupled d_out{ops::randn({2, 197, 192}, Dtype::f32, rng, 1e-2),
                         ops::randn({2, 197, 192}, Dtype::f32, rng, 1e-2)};
  const A::Coupled ro = ref_rev_forward(blk, in);
  const A::Coupled go = A::rev_forward(blk, in);
  report("rev_forward o1", rel(go.i1, ro.i1), 2e-2);
  report("rev_forward o2", rel(go.i2, ro.i2), 2e-2);
  const A::Coupled gi = A::rev_inverse(blk, go);  // round trip on the B200
  report("rev_inverse round trip i1", rel(gi.i1, in.i1), 1e-4);
  report("rev_inverse round trip i2", rel(gi.i2, in.i2), 1e-4);
  // reference backward: recompute from the output, G path before F path
  const MlpForward mg = mlp_forward(ro.i2, blk.g);
  const Tensor i1 = ops::sub(ro.i1, mg.y);
  const AttentionForward af = attention_forward(i1, blk.f);
  const MlpVjp vg = mlp_vjp(mg.cache, blk.g, d_out.i1);
  const Tensor d_i2 = ops::add(d_out.i2, vg.d_x);
  const AttentionVjp vf = attention_vjp(af.cache, blk.f, d_i2);
  const Tensor d_i1 = ops::add(d_out.i1, vf.d_x);
  auto [inp, d_inp, g] = A::rev_backward_local(blk, ro, d_out);
  // (o1, o2) come from the reference's CPU forward, so the B200's recompute of i1 differs
  // from it by the B200-vs-CPU G evaluation (bf16 operands), not by a round trip
  report("rev_backward_local i1 (vs reference recompute)", rel(inp.i1, i1), 2e-2);
  report("rev_backward_local i2 (vs reference input)", rel(inp.i2, in.i2), 2e-2);
  report("rev_backward_local d_i1", rel(d_inp.i1, d_i1), 2e-2);
  report("rev_backward_local d_i2", rel(d_inp.i2, d_i2), 2e-2);
  report("rev_backward_local d_w_qkv", rel(g.d_f.d_w_qkv, vf.d_params.d_w_qkv), 2e-2);
  report("rev_backward_local d_w1", rel(g.d_g.d_w1, vg.d_params.d_w1), 2e-2);
  report("rev_backward_local d_w2", rel(g.d_g.d_w2, vg.d_params.d_w2), 2e-2);
}

static void check_sgd_and_errors() {
  // single scalar param p, grad g, lr 0.1 -> p - 0.1 g
  const Tensor p = Tensor::from_values({1}, {1.5}, Dtype::f32);
  const Tensor g = Tensor::from_values({1}, {2.0}, Dtype::f32);
  const Tensor q = A::sgd_update(p, g, 0.1);
  const float want = 1.5f - 0.1f * 2.0f;
  report_bool("sgd_update scalar p - 0.1 g (bit-exact)", static_cast<float>(q.get(0)) == want);
  report_bool("sgd_update lr = 0 leaves p unchanged",
              bits_equal(A::sgd_update(p, g, 0.0), p));
  // the reference's exception classes come back out of the B200 path
  Rng rng(3, 1);
  const AttentionParams ap = attn_params(192, 3, std::nullopt, rng);
  bool shape = false, contract = false;
  try {
    A::attention_forward(ops::randn({2, 5, 128}, Dtype::f32, rng), ap);  // width mismatch
  } catch (const ShapeError&) {
    shape = true;
  }
  report_bool("width mismatch -> revprop::ShapeError", shape);
  try {
    const MlpParams mp = mlp_params(192, 768, rng);
    const A::MlpForwardB200 mf = A::mlp_forward(ops::randn({1, 4, 192}, Dtype::f32, rng), mp);
    A::attention_vjp(B::AttentionCache{mf.cache.c}, ap, ops::randn({1, 4, 192}, Dtype::f32, rng));
  } catch (const ContractError&) {
    contract = true;
  }
  report_bool("wrong cache -> revprop::ContractError", contract);
}

static void check_engines() {
  RpModelConfig c{};
  c.depth = 3;
  c.width = 192;
  c.heads = 3;
  c.hidden = 768;
  c.seq_len = 197;
  c.in_dim = 768;
  c.num_classes = 10;
  c.batch = 4;
  c.seed = 5;
  B::Model m(c);
  Rng rng(11, 2);
  B::Batch batch;
  const Tensor x = ops::randn({4, 197, 768}, Dtype::f32, rng);
  for (std::size_t i = 0; i < x.numel(); ++i) batch.inputs.push_back(static_cast<float>(x.get(i)));
  batch.labels = {1, 7, 3, 9};
  B::MemoryLedger ledger;
  auto [gr, sr] = B::step_reprop(m, batch, ledger);
  auto [gp, sp] = B::step_pareprop(m, batch, ledger);
  report_bool("step_pareprop == step_reprop (bit-exact)",
              gr.flat == gp.flat && sr.loss == sp.loss);
  report_bool("StepStats.blocks_processed == depth", sr.blocks_processed == 3 &&
                                                          sp.blocks_processed == 3);
  report_bool("ledger peak = PaReprop peak, live 0",
              ledger.peak_bytes() == sp.peak_activation_bytes && ledger.live_bytes() == 0 &&
                  sp.peak_activation_bytes > sr.peak_activation_bytes);
  report_bool("GradStore tensor table covers the model",
              gr.offsets.size() == 1 + 10 * 3 + 1 &&
                  gr.offsets.back() + gr.numels.back() == static_cast<std::int64_t>(gr.flat.size()));
  const std::vector<float> p0 = m.params();
  B::sgd_update(m, gr, 0.25);
  const std::vector<float> p1 = m.params();
  bool exact = p1.size() == p0.size();
  for (std::size_t i = 0; exact && i < p0.size(); ++i) {
    const volatile float prod = 0.25f * gr.flat[i];
    exact = p1[i] == p0[i] - prod;
  }
  report_bool("sgd_update(model, grads, lr) bit-exact", exact);
  auto [g2, s2] = B::step_reprop(m, batch, ledger);
  report_bool("loss after one SGD step is finite", std::isfinite(s2.loss));
}

int main() {
  try {
    check_attention("attention (full, hd 64)", 2, 197, 192, 3, std::nullopt);
    check_attention("attention (windows of 49, hd 32)", 2, 196, 128, 4, 49);
    check_mlp();
    check_revcore();
    check_sgd_and_errors();
    check_engines();
  } catch (const std::exception& e) {
    std::printf("exception: %s\n", e.what());
    return 2;
  }
  std::printf("%s: %d failure(s)\n", g_fail ? "ADAPTER FAIL" : "ADAPTER OK", g_fail);
  return g_fail ? 1 : 0;
}
