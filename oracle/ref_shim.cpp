// TEST INFRASTRUCTURE ONLY -- the CPU oracle. Never linked into the product library.
//
// extern "C" surface over the reference implementation, compiled in place from
// /root/reference/proj/core/src/{ops,layers}.cpp (see oracle/Makefile), plus a
// restatement of the SPEC-only modules on top of the reference's own Tensor / layers API:
//   revcore: rev_forward, rev_inverse, rev_backward_local
//   models: isotropic forward_full, loss_and_grad_head
//   engines: step_reprop, step_pareprop (two lanes + rendezvous), sgd
// The reference ships no code for these; every function cites the SPEC
// lines it follows. Used by tests/ to pin the numpy oracle and to generate the golden
// fixtures, and by bench.py --impl reference as the CPU baseline.
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <mutex>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "revprop/errors.hpp"
#include "revprop/layers.hpp"
#include "revprop/ledger.hpp"
#include "revprop/ops.hpp"
#include "revprop/rng.hpp"
#include "revprop/tensor.hpp"

using namespace revprop;

namespace {

thread_local std::string g_err;

int code_of(const std::exception& e) {
  if (dynamic_cast<const ShapeError*>(&e)) return 1;
  if (dynamic_cast<const ContractError*>(&e)) return 2;
  if (dynamic_cast<const ConfigError*>(&e)) return 3;
  if (dynamic_cast<const BudgetError*>(&e)) return 4;
  if (dynamic_cast<const SchedulerError*>(&e)) return 5;
  if (dynamic_cast<const AccountingError*>(&e)) return 6;
  return 7;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return code_of(e);
  }
}

Dtype dt_of(int f64) { return f64 ? Dtype::f64 : Dtype::f32; }

Tensor from_raw(const void* p, std::vector<std::size_t> dims, Dtype dt) {
  Tensor t = Tensor::zeros(std::move(dims), dt);
  if (dt == Dtype::f64)
    std::memcpy(t.values<double>().data(), p, t.byte_size());
  else
    std::memcpy(t.values<float>().data(), p, t.byte_size());
  return t;
}

void to_raw(const Tensor& t, void* p) {
  if (!p) return;
  if (t.dtype() == Dtype::f64)
    std::memcpy(p, t.values<double>().data(), t.byte_size());
  else
    std::memcpy(p, t.values<float>().data(), t.byte_size());
}

}  // namespace

extern "C" {

// Model geometry (isotropic RevViT / Rev-RoBERTa).
typedef struct {
  int64_t depth, width, heads, hidden, seq_len, in_dim, num_classes, window;  // window 0 = full
} RefCfg;

const char* ref_last_error(void) { return g_err.c_str(); }

}  // extern "C"

namespace {

// ---------------------------------------------------------------- parameter layout
// Flat order (shared with the GPU engine and the numpy oracle):
//   embed_w [in,d] | per block: w_qkv [d,3d], w_out [d,d], lnF_g [d], lnF_b [d],
//                    w1 [d,h], b1 [h], w2 [h,d], b2 [d], lnG_g [d], lnG_b [d] | head_w [d,C]
struct Layout {
  int64_t d, h, in, C, L;
  int64_t block_size() const { return 4 * d * d + 2 * d * h + h + 5 * d; }
  int64_t embed_off() const { return 0; }
  int64_t block_off(int64_t i) const { return in * d + i * block_size(); }
  int64_t head_off() const { return in * d + L * block_size(); }
  int64_t total() const { return head_off() + d * C; }
};

Layout layout_of(const RefCfg& c) {
  return Layout{c.width, c.hidden, c.in_dim, c.num_classes, c.depth};
}

struct View {
  const uint8_t* base;
  Dtype dt;
  Tensor take(int64_t& off, std::vector<std::size_t> dims) const {
    std::size_t n = 1;
    for (auto x : dims) n *= x;
    Tensor t = from_raw(base + off * static_cast<int64_t>(dtype_size(dt)), std::move(dims), dt);
    off += static_cast<int64_t>(n);
    return t;
  }
};

struct RevBlock {
  AttentionParams f;
  MlpParams g;
  int64_t id;
};

RevBlock block_from(const RefCfg& c, const void* p, Dtype dt, int64_t id) {
  const std::size_t d = c.width, h = c.hidden;
  View v{static_cast<const uint8_t*>(p), dt};
  int64_t off = 0;
  RevBlock b;
  b.f.w_qkv = v.take(off, {d, 3 * d});
  b.f.w_out = v.take(off, {d, d});
  b.f.ln_gamma = v.take(off, {d});
  b.f.ln_beta = v.take(off, {d});
  b.f.heads = static_cast<std::size_t>(c.heads);
  if (c.window > 0) b.f.window = static_cast<std::size_t>(c.window);
  b.g.w1 = v.take(off, {d, h});
  b.g.b1 = v.take(off, {h});
  b.g.w2 = v.take(off, {h, d});
  b.g.b2 = v.take(off, {d});
  b.g.ln_gamma = v.take(off, {d});
  b.g.ln_beta = v.take(off, {d});
  b.id = id;
  return b;
}

struct RevBlockGrads {
  AttentionGrads f;
  MlpGrads g;
};

void grads_to_raw(const RevBlockGrads& gr, void* out) {
  if (!out) return;
  uint8_t* p = static_cast<uint8_t*>(out);
  auto put = [&](const Tensor& t) {
    to_raw(t, p);
    p += t.byte_size();
  };
  put(gr.f.d_w_qkv);
  put(gr.f.d_w_out);
  put(gr.f.d_ln_gamma);
  put(gr.f.d_ln_beta);
  put(gr.g.d_w1);
  put(gr.g.d_b1);
  put(gr.g.d_w2);
  put(gr.g.d_b2);
  put(gr.g.d_ln_gamma);
  put(gr.g.d_ln_beta);
}

struct Coupled {
  Tensor i1, i2;
};

// rev_forward: o2 = i2 + F(i1); o1 = i1 + G(o2). Stores nothing.
Coupled rev_forward(const RevBlock& b, const Coupled& in) {
  Tensor o2 = ops::add(in.i2, attention_forward(in.i1, b.f).y);
  Tensor o1 = ops::add(in.i1, mlp_forward(o2, b.g).y);
  return Coupled{std::move(o1), std::move(o2)};
}

// rev_inverse: i1 = o1 - G(o2); i2 = o2 - F(i1). One F, one G call.
Coupled rev_inverse(const RevBlock& b, const Coupled& out) {
  Tensor i1 = ops::sub(out.i1, mlp_forward(out.i2, b.g).y);
  Tensor i2 = ops::sub(out.i2, attention_forward(i1, b.f).y);
  return Coupled{std::move(i1), std::move(i2)};
}

// Lane-R half of rev_backward_local: the inverse with F/G caches retained.
struct Recomputed {
  Coupled inp;
  AttentionCache cf;
  MlpCache cg;
  std::int64_t bytes() const {
    return static_cast<std::int64_t>(cf.byte_size() + cg.byte_size() + inp.i1.byte_size() +
                                     inp.i2.byte_size());
  }
};

Recomputed recompute(const RevBlock& b, const Coupled& out) {
  MlpForward g = mlp_forward(out.i2, b.g);
  Tensor i1 = ops::sub(out.i1, g.y);
  AttentionForward f = attention_forward(i1, b.f);
  Tensor i2 = ops::sub(out.i2, f.y);
  return Recomputed{Coupled{std::move(i1), std::move(i2)}, std::move(f.cache), std::move(g.cache)};
}

// First block of a stage: its input is the stored stage boundary, so the R slot runs
// F and G forward with caches from it (no subtraction) -- SURVEY.md §0 resolution of the
// SPEC.md:414 vs :385/:503 slot-count inconsistency.
Recomputed recompute_from_input(const RevBlock& b, const Coupled& inp) {
  AttentionForward f = attention_forward(inp.i1, b.f);
  Tensor o2 = ops::add(inp.i2, f.y);
  MlpForward g = mlp_forward(o2, b.g);
  return Recomputed{inp, std::move(f.cache), std::move(g.cache)};
}

// Lane-G half: d_o2t = d_o2 + VJP_G(d_o1); d_i1 = d_o1 + VJP_F(d_o2t);
// d_i2 = d_o2t. G-path before F-path. Caches die on return.
Coupled vjp_half(const RevBlock& b, const Recomputed& r, const Coupled& d_out,
                 RevBlockGrads& grads) {
  MlpVjp gv = mlp_vjp(r.cg, b.g, d_out.i1);
  Tensor d_o2t = ops::add(d_out.i2, gv.d_x);
  AttentionVjp fv = attention_vjp(r.cf, b.f, d_o2t);
  Tensor d_i1 = ops::add(d_out.i1, fv.d_x);
  grads.f = std::move(fv.d_params);
  grads.g = std::move(gv.d_params);
  return Coupled{std::move(d_i1), std::move(d_o2t)};
}

// ---------------------------------------------------------------- model glue
struct ModelView {
  RefCfg cfg;
  Layout lay;
  Dtype dt;
  Tensor embed_w, head_w;
  std::vector<RevBlock> blocks;
};

ModelView model_from(const RefCfg& c, const void* params, Dtype dt) {
  ModelView m{c, layout_of(c), dt, {}, {}, {}};
  View v{static_cast<const uint8_t*>(params), dt};
  int64_t off = 0;
  m.embed_w = v.take(off, {static_cast<std::size_t>(c.in_dim), static_cast<std::size_t>(c.width)});
  const int64_t esz = static_cast<int64_t>(dtype_size(dt));
  for (int64_t i = 0; i < c.depth; ++i)
    m.blocks.push_back(
        block_from(c, static_cast<const uint8_t*>(params) + m.lay.block_off(i) * esz, dt, i));
  off = m.lay.head_off();
  m.head_w = v.take(off, {static_cast<std::size_t>(c.width), static_cast<std::size_t>(c.num_classes)});
  return m;
}

// mean cross-entropy with log-sum-exp stabilisation; d_logits = (softmax - onehot)/B
// (SPEC.md:307-316).
double loss_and_grad_head(const Tensor& logits, const std::vector<int64_t>& labels,
                          Tensor& d_logits) {
  const std::size_t B = logits.dim(0), C = logits.dim(1);
  d_logits = Tensor::zeros_like(logits);
  double loss = 0.0;
  for (std::size_t b = 0; b < B; ++b) {
    if (labels[b] < 0 || static_cast<std::size_t>(labels[b]) >= C)
      throw ShapeError("loss: label out of range");
    double mx = logits.get(b * C);
    for (std::size_t c = 1; c < C; ++c) mx = std::max(mx, logits.get(b * C + c));
    double s = 0.0;
    for (std::size_t c = 0; c < C; ++c) s += std::exp(logits.get(b * C + c) - mx);
    const double lse = mx + std::log(s);
    loss += lse - logits.get(b * C + static_cast<std::size_t>(labels[b]));
    for (std::size_t c = 0; c < C; ++c) {
      const double p = std::exp(logits.get(b * C + c) - lse);
      d_logits.set(b * C + c, (p - (static_cast<int64_t>(c) == labels[b] ? 1.0 : 0.0)) /
                                  static_cast<double>(B));
    }
  }
  return loss / static_cast<double>(B);
}

struct SlotEvent {
  int lane;  // 0 = R (recompute), 1 = G (gradient)
  int64_t block;
  int64_t t0, t1;
};

struct StepOut {
  double loss = 0.0;
  std::vector<Tensor> grads;  // flat order: embed, blocks (10 each), head
  int64_t peak = 0;
  std::vector<SlotEvent> slots;
};

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// Rendezvous of capacity 1: lane R may start block i-1 only after
// lane G has taken block i, so at most two blocks' caches are live.
struct Rendezvous {
  std::mutex mu;
  std::condition_variable cv;
  std::optional<Recomputed> slot;
  bool failed = false;
  std::string why;
  void wait_empty() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return !slot.has_value() || failed; });
    if (failed) throw SchedulerError("pipeline lane failed: " + why);
  }
  void put(Recomputed r) {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return !slot.has_value() || failed; });
    if (failed) throw SchedulerError("pipeline lane failed: " + why);
    slot.emplace(std::move(r));
    cv.notify_all();
  }
  Recomputed take() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [&] { return slot.has_value() || failed; });
    if (failed) throw SchedulerError("pipeline lane failed: " + why);
    Recomputed r = std::move(*slot);
    slot.reset();
    cv.notify_all();
    return r;
  }
  void fail(const std::string& w) {
    std::lock_guard<std::mutex> lk(mu);
    failed = true;
    why = w;
    cv.notify_all();
  }
};

// step_reprop / step_pareprop.
StepOut run_step(const ModelView& m, const Tensor& inputs, const std::vector<int64_t>& labels,
                 bool pipelined, bool log_slots) {
  StepOut out;
  MemoryLedger ledger;
  const RefCfg& c = m.cfg;
  // ---- forward_full: embed, duplicate, blocks, fuse(avg), pool, head
  Tensor e = ops::matmul(inputs, m.embed_w);
  Coupled stage_in{e, e};
  LedgerCharge charge_in(&ledger, "stage_in",
                         static_cast<int64_t>(e.byte_size() * 2));
  Coupled x = stage_in;
  for (const RevBlock& b : m.blocks) x = rev_forward(b, x);
  LedgerCharge charge_out(&ledger, "stage_out", static_cast<int64_t>(x.i1.byte_size() * 2));
  BoundaryParams avg;
  FuseResult fused = fuse(x.i1, x.i2, avg);
  Tensor pooled = ops::mean_tokens(fused.y);
  Tensor logits = ops::matmul(pooled, m.head_w);
  Tensor d_logits;
  out.loss = loss_and_grad_head(logits, labels, d_logits);
  // ---- head backward
  Tensor d_head_w = ops::matmul_tn(pooled, d_logits);
  Tensor d_pooled = ops::matmul_nt(d_logits, m.head_w);
  Tensor d_fused = ops::spread_tokens(d_pooled, static_cast<std::size_t>(c.seq_len));
  FuseVjp fv = fuse_vjp(fused, avg, d_fused);
  Coupled d_out{std::move(fv.d_i1), std::move(fv.d_i2)};

  const int64_t L = c.depth;
  std::vector<RevBlockGrads> bgrads(static_cast<std::size_t>(L));
  std::mutex log_mu;
  auto log_slot = [&](int lane, int64_t blk, int64_t t0) {
    if (!log_slots) return;
    std::lock_guard<std::mutex> lk(log_mu);
    out.slots.push_back(SlotEvent{lane, blk + 1, t0, now_ns()});
  };
  auto do_r = [&](int64_t i, const Coupled& o) {
    const int64_t t0 = now_ns();
    Recomputed r = (i == 0) ? recompute_from_input(m.blocks[0], stage_in)
                            : recompute(m.blocks[static_cast<std::size_t>(i)], o);
    log_slot(0, i, t0);
    return r;
  };
  if (!pipelined) {
    Coupled o = x;
    for (int64_t i = L - 1; i >= 0; --i) {
      Recomputed r = do_r(i, o);
      LedgerCharge ch(&ledger, "block", r.bytes());
      const int64_t t0 = now_ns();
      d_out = vjp_half(m.blocks[static_cast<std::size_t>(i)], r, d_out,
                       bgrads[static_cast<std::size_t>(i)]);
      log_slot(1, i, t0);
      o = std::move(r.inp);
    }
  } else {
    Rendezvous rv;
    std::thread lane_r([&] {
      try {
        Coupled o = x;
        for (int64_t i = L - 1; i >= 0; --i) {
          rv.wait_empty();
          Recomputed r = do_r(i, o);
          ledger.track("block", r.bytes());
          o = r.inp;
          rv.put(std::move(r));
        }
      } catch (const std::exception& ex) {
        rv.fail(ex.what());
      }
    });
    try {
      for (int64_t i = L - 1; i >= 0; --i) {
        Recomputed r = rv.take();
        const int64_t t0 = now_ns();
        d_out = vjp_half(m.blocks[static_cast<std::size_t>(i)], r, d_out,
                         bgrads[static_cast<std::size_t>(i)]);
        log_slot(1, i, t0);
        ledger.track("block", -r.bytes());
      }
    } catch (const std::exception& ex) {
      rv.fail(ex.what());
      lane_r.join();
      throw SchedulerError(std::string("pipeline lane failed: ") + ex.what());
    }
    lane_r.join();
  }
  // ---- embedding backward: e feeds both i1 and i2 (duplication)
  Tensor d_e = ops::add(d_out.i1, d_out.i2);
  Tensor d_embed_w = ops::matmul_tn(inputs, d_e);
  out.grads.push_back(std::move(d_embed_w));
  for (auto& g : bgrads) {
    out.grads.push_back(std::move(g.f.d_w_qkv));
    out.grads.push_back(std::move(g.f.d_w_out));
    out.grads.push_back(std::move(g.f.d_ln_gamma));
    out.grads.push_back(std::move(g.f.d_ln_beta));
    out.grads.push_back(std::move(g.g.d_w1));
    out.grads.push_back(std::move(g.g.d_b1));
    out.grads.push_back(std::move(g.g.d_w2));
    out.grads.push_back(std::move(g.g.d_b2));
    out.grads.push_back(std::move(g.g.d_ln_gamma));
    out.grads.push_back(std::move(g.g.d_ln_beta));
  }
  out.grads.push_back(std::move(d_head_w));
  out.peak = ledger.peak_bytes();
  return out;
}

void flat_to_raw(const std::vector<Tensor>& ts, void* out) {
  uint8_t* p = static_cast<uint8_t*>(out);
  for (const Tensor& t : ts) {
    to_raw(t, p);
    p += t.byte_size();
  }
}

}  // namespace

extern "C" {

int64_t ref_param_count(const RefCfg* c) { return layout_of(*c).total(); }

// The reference counter RNG (rng.hpp:13-71), for pinning the vectorised restatement:
// n draws each of next_u64, next_normal and next_trunc_normal(1) from fresh Rng(seed, stream).
int ref_rng(uint64_t seed, uint64_t stream, int64_t n, uint64_t* u64_out, double* normal_out,
            double* trunc_out) {
  return guarded([&] {
    Rng a(seed, stream), b(seed, stream), c(seed, stream);
    for (int64_t i = 0; i < n; ++i) {
      if (u64_out) u64_out[i] = a.next_u64();
      if (normal_out) normal_out[i] = b.next_normal();
      if (trunc_out) trunc_out[i] = c.next_trunc_normal(1.0);
    }
  });
}
int64_t ref_block_param_count(const RefCfg* c) { return layout_of(*c).block_size(); }

// ops::layer_norm (ops.cpp:264-304) + layer_norm_vjp (ops.cpp:306-345)
int ref_layer_norm(int f64, const void* x, int64_t rows, int64_t cols, const void* g,
                   const void* b, double eps, const void* dy, void* y, void* inv_std, void* dx,
                   void* dg, void* db) {
  return guarded([&] {
    const Dtype dt = dt_of(f64);
    const std::size_t R = static_cast<std::size_t>(rows), Cc = static_cast<std::size_t>(cols);
    Tensor X = from_raw(x, {R, Cc}, dt), G = from_raw(g, {Cc}, dt), Bt = from_raw(b, {Cc}, dt);
    auto res = ops::layer_norm(X, G, Bt, eps);
    to_raw(res.y, y);
    to_raw(res.cache.inv_std, inv_std);
    if (dy) {
      auto v = ops::layer_norm_vjp(res.cache, G, from_raw(dy, {R, Cc}, dt));
      to_raw(v.d_x, dx);
      to_raw(v.d_gamma, dg);
      to_raw(v.d_beta, db);
    }
  });
}

// attention_forward + attention_vjp (layers.cpp:134-220) on block-F params
// [w_qkv | w_out | ln_g | ln_b]; d_params out in the same order.
int ref_attention(int f64, const RefCfg* c, int64_t B, const void* pf, const void* x,
                  const void* d_y, void* y, void* d_x, void* d_pf) {
  return guarded([&] {
    const Dtype dt = dt_of(f64);
    const std::size_t d = c->width;
    View v{static_cast<const uint8_t*>(pf), dt};
    int64_t off = 0;
    AttentionParams p;
    p.w_qkv = v.take(off, {d, 3 * d});
    p.w_out = v.take(off, {d, d});
    p.ln_gamma = v.take(off, {d});
    p.ln_beta = v.take(off, {d});
    p.heads = static_cast<std::size_t>(c->heads);
    if (c->window > 0) p.window = static_cast<std::size_t>(c->window);
    const std::vector<std::size_t> dims{static_cast<std::size_t>(B),
                                        static_cast<std::size_t>(c->seq_len), d};
    AttentionForward f = attention_forward(from_raw(x, dims, dt), p);
    to_raw(f.y, y);
    if (d_y) {
      AttentionVjp g = attention_vjp(f.cache, p, from_raw(d_y, dims, dt));
      to_raw(g.d_x, d_x);
      flat_to_raw({g.d_params.d_w_qkv, g.d_params.d_w_out, g.d_params.d_ln_gamma,
                   g.d_params.d_ln_beta},
                  d_pf);
    }
  });
}

// mlp_forward + mlp_vjp (layers.cpp:222-259) on block-G params [w1|b1|w2|b2|ln_g|ln_b]
int ref_mlp(int f64, const RefCfg* c, int64_t B, const void* pg, const void* x, const void* d_y,
            void* y, void* d_x, void* d_pg) {
  return guarded([&] {
    const Dtype dt = dt_of(f64);
    const std::size_t d = c->width, h = c->hidden;
    View v{static_cast<const uint8_t*>(pg), dt};
    int64_t off = 0;
    MlpParams p;
    p.w1 = v.take(off, {d, h});
    p.b1 = v.take(off, {h});
    p.w2 = v.take(off, {h, d});
    p.b2 = v.take(off, {d});
    p.ln_gamma = v.take(off, {d});
    p.ln_beta = v.take(off, {d});
    const std::vector<std::size_t> dims{static_cast<std::size_t>(B),
                                        static_cast<std::size_t>(c->seq_len), d};
    MlpForward f = mlp_forward(from_raw(x, dims, dt), p);
    to_raw(f.y, y);
    if (d_y) {
      MlpVjp g = mlp_vjp(f.cache, p, from_raw(d_y, dims, dt));
      to_raw(g.d_x, d_x);
      flat_to_raw({g.d_params.d_w1, g.d_params.d_b1, g.d_params.d_w2, g.d_params.d_b2,
                   g.d_params.d_ln_gamma, g.d_params.d_ln_beta},
                  d_pg);
    }
  });
}

int ref_rev_forward(int f64, const RefCfg* c, int64_t B, const void* pblock, const void* i1,
                    const void* i2, void* o1, void* o2) {
  return guarded([&] {
    const Dtype dt = dt_of(f64);
    const std::vector<std::size_t> dims{static_cast<std::size_t>(B),
                                        static_cast<std::size_t>(c->seq_len),
                                        static_cast<std::size_t>(c->width)};
    RevBlock b = block_from(*c, pblock, dt, 0);
    Coupled o = rev_forward(b, Coupled{from_raw(i1, dims, dt), from_raw(i2, dims, dt)});
    to_raw(o.i1, o1);
    to_raw(o.i2, o2);
  });
}

int ref_rev_inverse(int f64, const RefCfg* c, int64_t B, const void* pblock, const void* o1,
                    const void* o2, void* i1, void* i2) {
  return guarded([&] {
    const Dtype dt = dt_of(f64);
    const std::vector<std::size_t> dims{static_cast<std::size_t>(B),
                                        static_cast<std::size_t>(c->seq_len),
                                        static_cast<std::size_t>(c->width)};
    RevBlock b = block_from(*c, pblock, dt, 0);
    Coupled i = rev_inverse(b, Coupled{from_raw(o1, dims, dt), from_raw(o2, dims, dt)});
    to_raw(i.i1, i1);
    to_raw(i.i2, i2);
  });
}

// rev_backward_local
int ref_rev_backward_local(int f64, const RefCfg* c, int64_t B, const void* pblock,
                           const void* o1, const void* o2, const void* d_o1, const void* d_o2,
                           void* i1, void* i2, void* d_i1, void* d_i2, void* d_pblock) {
  return guarded([&] {
    const Dtype dt = dt_of(f64);
    const std::vector<std::size_t> dims{static_cast<std::size_t>(B),
                                        static_cast<std::size_t>(c->seq_len),
                                        static_cast<std::size_t>(c->width)};
    RevBlock b = block_from(*c, pblock, dt, 0);
    Recomputed r = recompute(b, Coupled{from_raw(o1, dims, dt), from_raw(o2, dims, dt)});
    RevBlockGrads g;
    Coupled di = vjp_half(b, r, Coupled{from_raw(d_o1, dims, dt), from_raw(d_o2, dims, dt)}, g);
    to_raw(r.inp.i1, i1);
    to_raw(r.inp.i2, i2);
    to_raw(di.i1, d_i1);
    to_raw(di.i2, d_i2);
    grads_to_raw(g, d_pblock);
  });
}

// One training step. engine: 1 = reprop, 2 = pareprop. grads: flat, parameter order.
// slots (optional): int64[4*2*depth] = (lane, block, t0, t1) per slot.
int ref_step(int f64, const RefCfg* c, int engine, int64_t B, const void* params,
             const void* inputs, const int64_t* labels, double* loss, void* grads,
             int64_t* peak_bytes, int64_t* slots) {
  return guarded([&] {
    if (engine != 1 && engine != 2) throw ConfigError("ref_step: engine must be 1 or 2");
    const Dtype dt = dt_of(f64);
    ModelView m = model_from(*c, params, dt);
    Tensor x = from_raw(inputs,
                        {static_cast<std::size_t>(B), static_cast<std::size_t>(c->seq_len),
                         static_cast<std::size_t>(c->in_dim)},
                        dt);
    std::vector<int64_t> lab(labels, labels + B);
    StepOut o = run_step(m, x, lab, engine == 2, slots != nullptr);
    if (loss) *loss = o.loss;
    if (grads) flat_to_raw(o.grads, grads);
    if (peak_bytes) *peak_bytes = o.peak;
    if (slots) {
      for (std::size_t i = 0; i < o.slots.size(); ++i) {
        slots[4 * i] = o.slots[i].lane;
        slots[4 * i + 1] = o.slots[i].block;
        slots[4 * i + 2] = o.slots[i].t0;
        slots[4 * i + 3] = o.slots[i].t1;
      }
    }
  });
}

// CPU baseline over all host threads: the batch is split into `threads` contiguous
// shards, each shard runs ref_step on its own thread, and the gradients are combined as
// sum_i (B_i/B) g_i (mean CE) in shard order. engine as in ref_step.
int ref_step_dp(int f64, const RefCfg* c, int engine, int64_t B, int threads,
                const void* params, const void* inputs, const int64_t* labels, double* loss,
                void* grads) {
  return guarded([&] {
    if (threads < 1) threads = 1;
    if (threads > B) threads = static_cast<int>(B);
    const Dtype dt = dt_of(f64);
    ModelView m = model_from(*c, params, dt);
    const std::size_t N = c->seq_len, in = c->in_dim;
    std::vector<StepOut> outs(static_cast<std::size_t>(threads));
    std::vector<int64_t> b0(threads + 1);
    for (int t = 0; t <= threads; ++t) b0[t] = B * t / threads;
    std::vector<std::string> errs(threads);
    std::vector<std::thread> ths;
    const std::size_t esz = dtype_size(dt);
    for (int t = 0; t < threads; ++t) {
      ths.emplace_back([&, t] {
        try {
          const int64_t nb = b0[t + 1] - b0[t];
          Tensor x = from_raw(static_cast<const uint8_t*>(inputs) + b0[t] * N * in * esz,
                              {static_cast<std::size_t>(nb), N, in}, dt);
          std::vector<int64_t> lab(labels + b0[t], labels + b0[t + 1]);
          outs[t] = run_step(m, x, lab, engine == 2, false);
        } catch (const std::exception& e) {
          errs[t] = e.what();
        }
      });
    }
    for (auto& th : ths) th.join();
    for (auto& e : errs)
      if (!e.empty()) throw SchedulerError("dp shard failed: " + e);
    double l = 0.0;
    std::vector<Tensor> acc;
    for (int t = 0; t < threads; ++t) {
      const double w = static_cast<double>(b0[t + 1] - b0[t]) / static_cast<double>(B);
      l += w * outs[t].loss;
      for (std::size_t k = 0; k < outs[t].grads.size(); ++k) {
        Tensor s = ops::scale(outs[t].grads[k], w);
        if (t == 0)
          acc.push_back(std::move(s));
        else
          ops::accumulate(acc[k], s);
      }
    }
    if (loss) *loss = l;
    if (grads) flat_to_raw(acc, grads);
  });
}


// ---------------------------------------------------------------- hierarchical model
// Rev-Swin-style model: stages of RevBlocks joined by the
// reference's own stage boundary (layers.cpp:261-303: fuse, then patch_merge, then the
// fused-and-merged tensor duplicated into the next stage's pair). Stage s has width
// widths[s], heads[s], MLP hidden ratio*widths[s], seq_len / r^s tokens and attention
// windows of min(window, tokens). Only each stage's input and output pair are stored; the
// backward recomputes the boundary's fuse from the stored stage output. Reprop order.
// Flat parameter order: embed_w | stage 0 blocks | merge_w_0 [, fusion_w_0] | stage 1
// blocks | ... | head_w (the numpy oracle's tensor_shapes and the GPU engine share it).
typedef struct {
  int64_t stages, depths[8], widths[8], heads[8], ratio, seq_len, in_dim, num_classes, window,
      reduction, fusion;  // fusion: 0 average, 1 mlp
} RefHierCfg;

int64_t ref_hier_param_count(const RefHierCfg* c) {
  int64_t n = c->in_dim * c->widths[0];
  for (int64_t s = 0; s < c->stages; ++s) {
    const int64_t d = c->widths[s], h = c->ratio * d;
    n += c->depths[s] * (4 * d * d + 2 * d * h + h + 5 * d);
    if (s + 1 < c->stages) n += c->reduction * d * c->widths[s + 1] + (c->fusion ? 2 * d * d : 0);
  }
  return n + c->widths[c->stages - 1] * c->num_classes;
}

int ref_hier_step(int f64, const RefHierCfg* c, int64_t B, const void* params,
                  const void* inputs, const int64_t* labels, double* loss, void* grads) {
  return guarded([&] {
    if (c->stages < 2 || c->stages > 8) throw ConfigError("ref_hier_step: 2..8 stages");
    const Dtype dt = dt_of(f64);
    const std::size_t esz = dtype_size(dt);
    const uint8_t* base = static_cast<const uint8_t*>(params);
    View v{base, dt};
    int64_t off = 0;
    const std::size_t S = static_cast<std::size_t>(c->stages);
    Tensor embed_w = v.take(off, {static_cast<std::size_t>(c->in_dim),
                                  static_cast<std::size_t>(c->widths[0])});
    std::vector<std::vector<RevBlock>> blocks(S);
    std::vector<BoundaryParams> bnd(S - 1);
    std::vector<int64_t> toks(S);
    int64_t n = c->seq_len;
    for (std::size_t s = 0; s < S; ++s) {
      if (s) {
        if (n % c->reduction) throw ShapeError("seq_len not divisible by r^(stages-1)");
        n /= c->reduction;
      }
      toks[s] = n;
      RefCfg sc{c->depths[s], c->widths[s], c->heads[s], c->ratio * c->widths[s], n, c->in_dim,
                c->num_classes, c->window > 0 ? std::min(c->window, n) : 0};
      const int64_t bs = layout_of(sc).block_size();
      for (int64_t i = 0; i < c->depths[s]; ++i) {
        blocks[s].push_back(block_from(sc, base + off * static_cast<int64_t>(esz), dt, i));
        off += bs;
      }
      if (s + 1 < S) {
        const std::size_t d = static_cast<std::size_t>(c->widths[s]);
        bnd[s].reduction = static_cast<std::size_t>(c->reduction);
        bnd[s].merge_w = v.take(off, {bnd[s].reduction * d, static_cast<std::size_t>(c->widths[s + 1])});
        if (c->fusion) {
          bnd[s].fusion_kind = FusionKind::mlp;
          bnd[s].fusion_w = v.take(off, {2 * d, d});
        }
      }
    }
    Tensor head_w = v.take(off, {static_cast<std::size_t>(c->widths[S - 1]),
                                 static_cast<std::size_t>(c->num_classes)});
    Tensor x = from_raw(inputs,
                        {static_cast<std::size_t>(B), static_cast<std::size_t>(c->seq_len),
                         static_cast<std::size_t>(c->in_dim)},
                        dt);
    // forward_full
    Tensor e = ops::matmul(x, embed_w);
    std::vector<Coupled> s_in, s_out;
    Coupled cur{e, e};
    for (std::size_t s = 0; s < S; ++s) {
      s_in.push_back(cur);
      for (const RevBlock& b : blocks[s]) cur = rev_forward(b, cur);
      s_out.push_back(cur);
      if (s + 1 < S) {
        FuseResult f = fuse(cur.i1, cur.i2, bnd[s]);
        PatchMergeResult pm = patch_merge(f.y, bnd[s]);
        cur = Coupled{pm.y, pm.y};
      }
    }
    BoundaryParams avg;
    FuseResult fused = fuse(cur.i1, cur.i2, avg);
    Tensor pooled = ops::mean_tokens(fused.y);
    Tensor logits = ops::matmul(pooled, head_w);
    Tensor d_logits;
    std::vector<int64_t> lab(labels, labels + B);
    const double l = loss_and_grad_head(logits, lab, d_logits);
    Tensor d_head_w = ops::matmul_tn(pooled, d_logits);
    Tensor d_pooled = ops::matmul_nt(d_logits, head_w);
    FuseVjp fv0 = fuse_vjp(fused, avg,
                           ops::spread_tokens(d_pooled, static_cast<std::size_t>(toks[S - 1])));
    Coupled d_out{std::move(fv0.d_i1), std::move(fv0.d_i2)};
    std::vector<std::vector<RevBlockGrads>> bg(S);
    std::vector<Tensor> d_merge(S - 1), d_fusion(S - 1);
    for (std::size_t s = S; s-- > 0;) {
      const std::size_t L = blocks[s].size();
      bg[s].resize(L);
      Coupled o = s_out[s];
      for (std::size_t i = L; i-- > 0;) {
        Recomputed r = i == 0 ? recompute_from_input(blocks[s][0], s_in[s])
                              : recompute(blocks[s][i], o);
        d_out = vjp_half(blocks[s][i], r, d_out, bg[s][i]);
        o = std::move(r.inp);
      }
      if (s > 0) {
        Tensor d_y = ops::add(d_out.i1, d_out.i2);
        FuseResult f = fuse(s_out[s - 1].i1, s_out[s - 1].i2, bnd[s - 1]);
        PatchMergeResult pm = patch_merge(f.y, bnd[s - 1]);
        PatchMergeVjp pv = patch_merge_vjp(pm.grouped, bnd[s - 1], d_y);
        d_merge[s - 1] = std::move(pv.d_merge_w);
        FuseVjp fv = fuse_vjp(f, bnd[s - 1], pv.d_x);
        if (fv.d_fusion_w) d_fusion[s - 1] = std::move(*fv.d_fusion_w);
        d_out = Coupled{std::move(fv.d_i1), std::move(fv.d_i2)};
      }
    }
    Tensor d_embed_w = ops::matmul_tn(x, ops::add(d_out.i1, d_out.i2));
    if (loss) *loss = l;
    if (!grads) return;
    std::vector<Tensor> out;
    out.push_back(std::move(d_embed_w));
    for (std::size_t s = 0; s < S; ++s) {
      for (auto& g : bg[s]) {
        for (Tensor* t : {&g.f.d_w_qkv, &g.f.d_w_out, &g.f.d_ln_gamma, &g.f.d_ln_beta, &g.g.d_w1,
                          &g.g.d_b1, &g.g.d_w2, &g.g.d_b2, &g.g.d_ln_gamma, &g.g.d_ln_beta})
          out.push_back(std::move(*t));
      }
      if (s + 1 < S) {
        out.push_back(std::move(d_merge[s]));
        if (c->fusion) out.push_back(std::move(d_fusion[s]));
      }
    }
    out.push_back(std::move(d_head_w));
    flat_to_raw(out, grads);
  });
}

// The reference's boundary layers on raw arrays (layers.cpp:261-303): y = patch_merge(
// fuse(i1, i2)) and, given d_y, the cotangents d_i1, d_i2, d_merge_w, d_fusion_w.
int ref_boundary(int f64, int64_t B, int64_t N, int64_t d, int64_t d_next, int64_t r, int fusion,
                 const void* i1, const void* i2, const void* merge_w, const void* fusion_w,
                 const void* d_y, void* y, void* d_i1, void* d_i2, void* d_merge_w,
                 void* d_fusion_w) {
  return guarded([&] {
    const Dtype dt = dt_of(f64);
    const std::size_t b = B, n = N, dd = d, dn = d_next, rr = r;
    Tensor a = from_raw(i1, {b, n, dd}, dt), c = from_raw(i2, {b, n, dd}, dt);
    BoundaryParams p;
    p.reduction = rr;
    p.merge_w = from_raw(merge_w, {rr * dd, dn}, dt);
    if (fusion) {
      p.fusion_kind = FusionKind::mlp;
      p.fusion_w = from_raw(fusion_w, {2 * dd, dd}, dt);
    }
    FuseResult f = fuse(a, c, p);
    PatchMergeResult pm = patch_merge(f.y, p);
    to_raw(pm.y, y);
    if (!d_y) return;
    PatchMergeVjp pv = patch_merge_vjp(pm.grouped, p, from_raw(d_y, {b, n / rr, dn}, dt));
    FuseVjp fv = fuse_vjp(f, p, pv.d_x);
    to_raw(fv.d_i1, d_i1);
    to_raw(fv.d_i2, d_i2);
    to_raw(pv.d_merge_w, d_merge_w);
    if (fv.d_fusion_w) to_raw(*fv.d_fusion_w, d_fusion_w);
  });
}

}  // extern "C"
