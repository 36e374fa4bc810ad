// revprop_b200.hpp -- the reference's C++ API for the reversible training path, on B200.
//
// Header-only C++17 wrapper over the C ABI (revprop_b200.h). It keeps the reference's names,
// struct shapes and error behaviour so a caller of the reference switches over by changing
// a namespace and moving tensors to the device:
//
//   reference (ref:proj/core/include/revprop/layers.hpp, SPEC.md revcore / engines)
//     revprop::attention_forward(const Tensor&, const AttentionParams&) -> AttentionForward
//     revprop::attention_vjp(const AttentionCache&, const AttentionParams&, const Tensor&)
//     revprop::mlp_forward / mlp_vjp                                  (layers.hpp:131, 138)
//     rev_forward / rev_inverse / rev_backward_local(RevBlock, Coupled, ...)
//     step_reprop / step_pareprop / step_vanilla(Model&, Batch, MemoryLedger&)
//     sgd_update(model, grads, lr)
//   here: the same names in namespace revprop::b200, over DeviceTensor (fp32, device
//   memory, same dims and row-major layout as the reference's Tensor).
//
// Errors are the reference's exception classes (errors.hpp:9-48): when the reference's
// include tree is on the include path its own revprop::ShapeError etc. are thrown;
// otherwise this header declares the identical hierarchy in namespace revprop.
//
// Calls are synchronous with respect to the host (like the reference's value-returning
// functions): results are complete on return. Work runs on the calling thread's legacy
// default stream unless set_stream() picks another.
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "revprop_b200.h"

#if defined(__has_include)
#if __has_include("revprop/errors.hpp")
#include "revprop/errors.hpp"
#define REVPROP_B200_REFERENCE_ERRORS 1
#endif
#endif

#ifndef REVPROP_B200_REFERENCE_ERRORS
#include <stdexcept>
namespace revprop {
// identical to ref:proj/core/include/revprop/errors.hpp:9-48
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class ShapeError : public Error {
 public:
  explicit ShapeError(const std::string& what) : Error(what) {}
};
class ContractError : public Error {
 public:
  explicit ContractError(const std::string& what) : Error(what) {}
};
class ConfigError : public Error {
 public:
  explicit ConfigError(const std::string& what) : Error(what) {}
};
class BudgetError : public Error {
 public:
  explicit BudgetError(const std::string& what) : Error(what) {}
};
class SchedulerError : public Error {
 public:
  explicit SchedulerError(const std::string& what) : Error(what) {}
};
class AccountingError : public Error {
 public:
  explicit AccountingError(const std::string& what) : Error(what) {}
};
}  // namespace revprop
#endif

namespace revprop::b200 {

// ---------------------------------------------------------------- errors and streams
/// Status code -> the reference's exception class (revprop_b200.h status table).
inline void check(int rc, const char* what = "") {
  if (rc == RP_OK) return;
  const std::string m = std::string(what) + (what[0] ? ": " : "") + rp_last_error();
  switch (rc) {
    case RP_ERR_SHAPE: throw ShapeError(m);
    case RP_ERR_CONTRACT: throw ContractError(m);
    case RP_ERR_CONFIG: throw ConfigError(m);
    case RP_ERR_BUDGET: throw BudgetError(m);
    case RP_ERR_SCHEDULER: throw SchedulerError(m);
    case RP_ERR_ACCOUNTING: throw AccountingError(m);
    default: throw Error(m);
  }
}
inline void check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  const std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  if (e == cudaErrorMemoryAllocation) throw BudgetError(m);
  throw Error(m);
}

inline cudaStream_t& current_stream() {
  static thread_local cudaStream_t s = nullptr;  // legacy default stream
  return s;
}
/// Stream the following calls of this thread enqueue on (they still return complete).
inline void set_stream(cudaStream_t s) { current_stream() = s; }
inline void sync() { check_cuda(cudaStreamSynchronize(current_stream()), "stream"); }

// ---------------------------------------------------------------- DeviceTensor
/// Dense fp32 array in device memory, row-major, with the reference Tensor's dims
/// (tensor.hpp:13-135). Value semantics: copies are deep (device to device).
class DeviceTensor {
 public:
  DeviceTensor() = default;
  static DeviceTensor zeros(std::vector<std::size_t> dims) {
    DeviceTensor t;
    t.dims_ = std::move(dims);
    t.alloc();
    if (t.numel())
      check_cuda(cudaMemsetAsync(t.p_.get(), 0, t.byte_size(), current_stream()), "memset");
    return t;
  }
  static DeviceTensor from_host(std::vector<std::size_t> dims, const float* host) {
    DeviceTensor t;
    t.dims_ = std::move(dims);
    t.alloc();
    if (t.numel())
      check_cuda(cudaMemcpy(t.p_.get(), host, t.byte_size(), cudaMemcpyHostToDevice), "upload");
    return t;
  }
  static DeviceTensor from_host(std::vector<std::size_t> dims, const std::vector<float>& host) {
    DeviceTensor t;
    t.dims_ = std::move(dims);
    if (host.size() != t.numel())
      throw ShapeError("from_host: " + std::to_string(host.size()) + " values for " +
                       std::to_string(t.numel()) + " elements");
    return from_host(t.dims_, host.data());
  }
  DeviceTensor(const DeviceTensor& o) : dims_(o.dims_) {
    alloc();
    if (numel()) {
      check_cuda(cudaMemcpyAsync(p_.get(), o.p_.get(), byte_size(), cudaMemcpyDeviceToDevice,
                                 current_stream()), "copy");
      sync();
    }
  }
  DeviceTensor& operator=(const DeviceTensor& o) {
    if (this != &o) *this = DeviceTensor(o);
    return *this;
  }
  DeviceTensor(DeviceTensor&&) noexcept = default;
  DeviceTensor& operator=(DeviceTensor&&) noexcept = default;

  std::vector<float> to_host() const {
    std::vector<float> h(numel());
    sync();
    if (numel()) check_cuda(cudaMemcpy(h.data(), p_.get(), byte_size(), cudaMemcpyDeviceToHost), "download");
    return h;
  }
  const std::vector<std::size_t>& dims() const { return dims_; }
  std::size_t rank() const { return dims_.size(); }
  std::size_t dim(std::size_t i) const { return dims_.at(i); }
  std::size_t numel() const {
    std::size_t n = dims_.empty() ? 0 : 1;
    for (std::size_t d : dims_) n *= d;
    return n;
  }
  std::size_t byte_size() const { return numel() * sizeof(float); }
  bool defined() const { return !dims_.empty(); }
  float* data() { return p_.get(); }
  const float* data() const { return p_.get(); }
  bool same_shape(const DeviceTensor& o) const { return dims_ == o.dims_; }

 private:
  struct Free {
    void operator()(float* p) const { cudaFree(p); }
  };
  void alloc() {
    void* q = nullptr;
    if (numel()) check_cuda(cudaMalloc(&q, byte_size()), "device allocation");
    p_.reset(static_cast<float*>(q));
  }
  std::vector<std::size_t> dims_;
  std::unique_ptr<float, Free> p_;
};

namespace detail {
struct CacheFree {
  void operator()(RpLayerCache* c) const { rp_layer_cache_destroy(c); }
};
using CachePtr = std::shared_ptr<RpLayerCache>;
inline void need(bool ok, const std::string& msg) {
  if (!ok) throw ShapeError(msg);
}
// [B, N, d] (or [N, d] = one sequence) -> (B, N)
inline std::pair<int64_t, int64_t> rows_of(const DeviceTensor& x, std::size_t d, const char* who) {
  need(x.rank() >= 2 && x.dims().back() == d,
       std::string(who) + ": input last dim must equal the model width");
  const int64_t N = static_cast<int64_t>(x.dim(x.rank() - 2));
  return {static_cast<int64_t>(x.numel() / (static_cast<std::size_t>(N) * d)), N};
}
}  // namespace detail

// ---------------------------------------------------------------- attention (F)
struct AttentionParams {  // layers.hpp:43-52
  DeviceTensor w_qkv;     // [d, 3d], no bias
  DeviceTensor w_out;     // [d, d], no bias
  DeviceTensor ln_gamma;  // [d]
  DeviceTensor ln_beta;   // [d]
  std::size_t heads = 1;
  std::optional<std::size_t> window;  // tokens per attention window; unset = full
  std::size_t width() const { return w_qkv.dim(0); }

  RpAttentionParamsDev dev() const {
    detail::need(w_qkv.rank() == 2 && w_qkv.dim(1) == 3 * width() && w_out.rank() == 2 &&
                     w_out.dim(0) == width() && w_out.dim(1) == width() &&
                     ln_gamma.numel() == width() && ln_beta.numel() == width(),
                 "AttentionParams: inconsistent shapes");
    return {w_qkv.data(), w_out.data(), ln_gamma.data(), ln_beta.data(),
            static_cast<int64_t>(width()), static_cast<int64_t>(heads),
            window ? static_cast<int64_t>(*window) : 0};
  }
};
/// AttentionCache (layers.hpp:54-65): opaque device buffers of the forward.
struct AttentionCache {
  detail::CachePtr c;
  std::size_t byte_size() const { return c ? static_cast<std::size_t>(rp_layer_cache_bytes(c.get())) : 0; }
};
struct AttentionGrads {  // layers.hpp:67-72
  DeviceTensor d_w_qkv, d_w_out, d_ln_gamma, d_ln_beta;
};
struct AttentionForward {
  DeviceTensor y;
  AttentionCache cache;
};
struct AttentionVjp {
  DeviceTensor d_x;
  AttentionGrads d_params;
};

inline AttentionForward attention_forward(const DeviceTensor& x, const AttentionParams& p) {
  const auto dp = p.dev();
  const auto [B, N] = detail::rows_of(x, p.width(), "attention_forward");
  AttentionForward r{DeviceTensor::zeros(x.dims()), {}};
  RpLayerCache* c = nullptr;
  check(rp_attention_forward(&dp, x.data(), B, N, r.y.data(), &c, current_stream()),
        "attention_forward");
  r.cache.c = detail::CachePtr(c, detail::CacheFree{});
  sync();
  return r;
}

inline AttentionVjp attention_vjp(const AttentionCache& cache, const AttentionParams& p,
                                  const DeviceTensor& d_y) {
  const auto dp = p.dev();
  const std::size_t d = p.width();
  AttentionVjp r{DeviceTensor::zeros(d_y.dims()),
                 {DeviceTensor::zeros({d, 3 * d}), DeviceTensor::zeros({d, d}),
                  DeviceTensor::zeros({d}), DeviceTensor::zeros({d})}};
  RpAttentionGradsDev g{r.d_params.d_w_qkv.data(), r.d_params.d_w_out.data(),
                        r.d_params.d_ln_gamma.data(), r.d_params.d_ln_beta.data()};
  check(rp_attention_vjp(cache.c.get(), &dp, d_y.data(), r.d_x.data(), &g, current_stream()),
        "attention_vjp");
  sync();
  return r;
}

// ---------------------------------------------------------------- MLP (G)
struct MlpParams {  // layers.hpp:94-103
  DeviceTensor w1;        // [d, h]
  DeviceTensor b1;        // [h]
  DeviceTensor w2;        // [h, d]
  DeviceTensor b2;        // [d]
  DeviceTensor ln_gamma;  // [d]
  DeviceTensor ln_beta;   // [d]
  std::size_t width() const { return w1.dim(0); }

  RpMlpParamsDev dev() const {
    detail::need(w1.rank() == 2 && w2.rank() == 2 && w2.dim(0) == w1.dim(1) &&
                     w2.dim(1) == width() && b1.numel() == w1.dim(1) && b2.numel() == width() &&
                     ln_gamma.numel() == width() && ln_beta.numel() == width(),
                 "MlpParams: inconsistent shapes");
    return {w1.data(), b1.data(), w2.data(), b2.data(), ln_gamma.data(), ln_beta.data(),
            static_cast<int64_t>(width()), static_cast<int64_t>(w1.dim(1))};
  }
};
struct MlpCache {  // layers.hpp:105-114
  detail::CachePtr c;
  std::size_t byte_size() const { return c ? static_cast<std::size_t>(rp_layer_cache_bytes(c.get())) : 0; }
};
struct MlpGrads {  // layers.hpp:116-123
  DeviceTensor d_w1, d_b1, d_w2, d_b2, d_ln_gamma, d_ln_beta;
};
struct MlpForward {
  DeviceTensor y;
  MlpCache cache;
};
struct MlpVjp {
  DeviceTensor d_x;
  MlpGrads d_params;
};

inline MlpForward mlp_forward(const DeviceTensor& x, const MlpParams& p) {
  const auto dp = p.dev();
  const auto [B, N] = detail::rows_of(x, p.width(), "mlp_forward");
  MlpForward r{DeviceTensor::zeros(x.dims()), {}};
  RpLayerCache* c = nullptr;
  check(rp_mlp_forward(&dp, x.data(), B, N, r.y.data(), &c, current_stream()), "mlp_forward");
  r.cache.c = detail::CachePtr(c, detail::CacheFree{});
  sync();
  return r;
}

inline MlpVjp mlp_vjp(const MlpCache& cache, const MlpParams& p, const DeviceTensor& d_y) {
  const auto dp = p.dev();
  const std::size_t d = p.width(), h = p.w1.dim(1);
  MlpVjp r{DeviceTensor::zeros(d_y.dims()),
           {DeviceTensor::zeros({d, h}), DeviceTensor::zeros({h}), DeviceTensor::zeros({h, d}),
            DeviceTensor::zeros({d}), DeviceTensor::zeros({d}), DeviceTensor::zeros({d})}};
  RpMlpGradsDev g{r.d_params.d_w1.data(), r.d_params.d_b1.data(), r.d_params.d_w2.data(),
                  r.d_params.d_b2.data(), r.d_params.d_ln_gamma.data(),
                  r.d_params.d_ln_beta.data()};
  check(rp_mlp_vjp(cache.c.get(), &dp, d_y.data(), r.d_x.data(), &g, current_stream()), "mlp_vjp");
  sync();
  return r;
}

// ---------------------------------------------------------------- revcore
struct Coupled {
  DeviceTensor i1, i2;
};
struct RevBlock {
  AttentionParams f;
  MlpParams g;
  std::size_t block_id = 0;
  RpRevBlockDev dev() const {
    detail::need(f.width() == g.width(), "RevBlock: F and G disagree on the model width");
    return {f.dev(), g.dev()};
  }
};
struct RevBlockGrads {
  AttentionGrads d_f;
  MlpGrads d_g;
};

namespace detail {
inline std::pair<int64_t, int64_t> pair_rows(const Coupled& c, std::size_t d, const char* who) {
  need(c.i1.same_shape(c.i2), std::string(who) + ": i1.dims != i2.dims");
  return rows_of(c.i1, d, who);
}
}  // namespace detail

/// o2 = i2 + F(i1); o1 = i1 + G(o2); returns (o1, o2) as Coupled{i1 = o1, i2 = o2}.
inline Coupled rev_forward(const RevBlock& b, const Coupled& inp) {
  const auto db = b.dev();
  const auto [B, N] = detail::pair_rows(inp, b.f.width(), "rev_forward");
  Coupled out{DeviceTensor::zeros(inp.i1.dims()), DeviceTensor::zeros(inp.i1.dims())};
  check(rp_rev_forward(&db, B, N, inp.i1.data(), inp.i2.data(), out.i1.data(), out.i2.data(),
                       current_stream()), "rev_forward");
  sync();
  return out;
}

/// i1 = o1 - G(o2); i2 = o2 - F(i1) (one F and one G evaluation).
inline Coupled rev_inverse(const RevBlock& b, const Coupled& out) {
  const auto db = b.dev();
  const auto [B, N] = detail::pair_rows(out, b.f.width(), "rev_inverse");
  Coupled inp{DeviceTensor::zeros(out.i1.dims()), DeviceTensor::zeros(out.i1.dims())};
  check(rp_rev_inverse(&db, B, N, out.i1.data(), out.i2.data(), inp.i1.data(), inp.i2.data(),
                       current_stream()), "rev_inverse");
  sync();
  return inp;
}

/// Recompute (i1, i2) from (o1, o2) and back-propagate (d_o1, d_o2): returns
/// (inp, d_inp, grads); G path before F path, caches released on return.
inline std::tuple<Coupled, Coupled, RevBlockGrads> rev_backward_local(const RevBlock& b,
                                                                      const Coupled& out,
                                                                      const Coupled& d_out) {
  const auto db = b.dev();
  const auto [B, N] = detail::pair_rows(out, b.f.width(), "rev_backward_local");
  detail::need(d_out.i1.same_shape(out.i1) && d_out.i2.same_shape(out.i2),
               "rev_backward_local: d_out shapes must match out");
  const std::size_t d = b.f.width(), h = b.g.w1.dim(1);
  const auto& dims = out.i1.dims();
  Coupled inp{DeviceTensor::zeros(dims), DeviceTensor::zeros(dims)};
  Coupled d_inp{DeviceTensor::zeros(dims), DeviceTensor::zeros(dims)};
  RevBlockGrads g{{DeviceTensor::zeros({d, 3 * d}), DeviceTensor::zeros({d, d}),
                   DeviceTensor::zeros({d}), DeviceTensor::zeros({d})},
                  {DeviceTensor::zeros({d, h}), DeviceTensor::zeros({h}),
                   DeviceTensor::zeros({h, d}), DeviceTensor::zeros({d}),
                   DeviceTensor::zeros({d}), DeviceTensor::zeros({d})}};
  RpRevBlockGradsDev gd{{g.d_f.d_w_qkv.data(), g.d_f.d_w_out.data(), g.d_f.d_ln_gamma.data(),
                         g.d_f.d_ln_beta.data()},
                        {g.d_g.d_w1.data(), g.d_g.d_b1.data(), g.d_g.d_w2.data(),
                         g.d_g.d_b2.data(), g.d_g.d_ln_gamma.data(), g.d_g.d_ln_beta.data()}};
  check(rp_rev_backward_local(&db, B, N, out.i1.data(), out.i2.data(), d_out.i1.data(),
                              d_out.i2.data(), inp.i1.data(), inp.i2.data(), d_inp.i1.data(),
                              d_inp.i2.data(), &gd, current_stream()),
        "rev_backward_local");
  sync();
  return {std::move(inp), std::move(d_inp), std::move(g)};
}

/// theta <- theta - lr * g on one tensor (bit-identical to fp32 p - lr*g).
inline void sgd_update(DeviceTensor& param, const DeviceTensor& grad, double lr) {
  if (!param.same_shape(grad)) throw ContractError("sgd_update: missing or mismatched grads");
  check(rp_sgd_update(param.data(), grad.data(), static_cast<int64_t>(param.numel()),
                      static_cast<float>(lr), current_stream()), "sgd_update");
  sync();
}
/// every parameter of a block.
inline RevBlock sgd_update(const RevBlock& b, const RevBlockGrads& g, double lr) {
  RevBlock r = b;
  sgd_update(r.f.w_qkv, g.d_f.d_w_qkv, lr);
  sgd_update(r.f.w_out, g.d_f.d_w_out, lr);
  sgd_update(r.f.ln_gamma, g.d_f.d_ln_gamma, lr);
  sgd_update(r.f.ln_beta, g.d_f.d_ln_beta, lr);
  sgd_update(r.g.w1, g.d_g.d_w1, lr);
  sgd_update(r.g.b1, g.d_g.d_b1, lr);
  sgd_update(r.g.w2, g.d_g.d_w2, lr);
  sgd_update(r.g.b2, g.d_g.d_b2, lr);
  sgd_update(r.g.ln_gamma, g.d_g.d_ln_gamma, lr);
  sgd_update(r.g.ln_beta, g.d_g.d_ln_beta, lr);
  return r;
}

// ---------------------------------------------------------------- engines
/// MemoryLedger (ledger.hpp:18-104): the engine reports each step's activation peak and its
/// ledger event count; live bytes return to zero at the end of every step.
class MemoryLedger {
 public:
  void track(std::int64_t delta) {
    if (live_ + delta < 0) throw AccountingError("ledger underflow");
    live_ += delta;
    if (live_ > peak_) peak_ = live_;
    ++events_;
  }
  std::int64_t live_bytes() const { return live_; }
  std::int64_t peak_bytes() const { return peak_; }
  std::int64_t events() const { return events_; }
  void reset() { live_ = peak_ = events_ = 0; }

 private:
  std::int64_t live_ = 0, peak_ = 0, events_ = 0;
};

struct StepStats {
  double loss = 0.0;
  std::int64_t wall_ns = 0;
  std::int64_t peak_activation_bytes = 0;
  std::int64_t lane_busy_ns[2] = {-1, -1};
  std::int64_t blocks_processed = 0;
};

/// GradStore: the flat gradient vector (mean over data-parallel ranks) and
/// the tensor table in the engine's parameter order (revprop_b200.h).
struct GradStore {
  std::vector<float> flat;
  std::vector<std::int64_t> offsets, numels;
  std::vector<float> tensor(std::size_t i) const {
    return {flat.begin() + offsets.at(i), flat.begin() + offsets.at(i) + numels.at(i)};
  }
};

struct Batch {  // inputs [B, N, in_dim], labels in [0, C)
  std::vector<float> inputs;
  std::vector<std::int32_t> labels;
};

/// The model lives on the device inside an engine (parameters, arena, streams, graphs).
class Model {
 public:
  explicit Model(const RpModelConfig& cfg) : cfg_(cfg) {
    RpEngine* e = nullptr;
    check(rp_engine_create(&cfg, &e), "engine_create");
    e_.reset(e);
    check(rp_engine_set_lr(e, 0.f), "set_lr");  // steps compute grads; sgd_update applies them
  }
  RpEngine* engine() const { return e_.get(); }
  const RpModelConfig& config() const { return cfg_; }
  std::int64_t param_count() const { return rp_engine_param_count(e_.get()); }
  std::vector<float> params() const {
    std::vector<float> h(static_cast<std::size_t>(param_count()));
    check(rp_engine_get_params(e_.get(), h.data()), "get_params");
    return h;
  }
  void set_params(const std::vector<float>& h) {
    if (static_cast<std::int64_t>(h.size()) != param_count()) throw ShapeError("set_params: size");
    check(rp_engine_set_params(e_.get(), h.data()), "set_params");
  }

 private:
  struct Destroy {
    void operator()(RpEngine* e) const { rp_engine_destroy(e); }
  };
  RpModelConfig cfg_;
  std::unique_ptr<RpEngine, Destroy> e_;
};

namespace detail {
inline std::pair<GradStore, StepStats> run_step(Model& m, const Batch& batch, MemoryLedger& ledger,
                                                int mode) {
  const RpModelConfig& c = m.config();
  const std::size_t n = static_cast<std::size_t>(c.batch * c.seq_len * c.in_dim);
  if (batch.inputs.size() != n || batch.labels.size() != static_cast<std::size_t>(c.batch))
    throw ShapeError("step: batch shape does not match the model config");
  for (std::int32_t l : batch.labels)
    if (l < 0 || l >= c.num_classes) throw ShapeError("step: label out of range");
  std::vector<std::uint16_t> xb(n);
  for (std::size_t i = 0; i < n; ++i) {  // round to nearest even bf16 (the GEMM operand)
    std::uint32_t u;
    std::memcpy(&u, &batch.inputs[i], 4);
    xb[i] = static_cast<std::uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
  }
  check(rp_engine_set_batch(m.engine(), xb.data(), batch.labels.data()), "set_batch");
  if (mode == 0) check(rp_engine_enable_vanilla(m.engine()), "enable_vanilla");
  check(rp_engine_step(m.engine(), mode, 1), "step");
  RpStepStats st{};
  check(rp_engine_step_stats(m.engine(), &st), "step_stats");
  std::pair<GradStore, StepStats> r;
  r.second.loss = st.loss;
  r.second.wall_ns = st.wall_ns;
  r.second.peak_activation_bytes = st.peak_activation_bytes;
  r.second.lane_busy_ns[0] = st.lane_busy_ns[0];
  r.second.lane_busy_ns[1] = st.lane_busy_ns[1];
  r.second.blocks_processed = st.blocks_processed;
  ledger.track(st.peak_activation_bytes);  // the step's peak, released at its end
  ledger.track(-st.peak_activation_bytes);
  GradStore& g = r.first;
  g.flat.resize(static_cast<std::size_t>(m.param_count()));
  check(rp_engine_get_grads(m.engine(), g.flat.data()), "get_grads");
  const std::int64_t cap = 16 + 10 * c.depth + 2 * 8;
  g.offsets.resize(static_cast<std::size_t>(cap));
  g.numels.resize(static_cast<std::size_t>(cap));
  const int k = rp_engine_tensor_table(m.engine(), g.offsets.data(), g.numels.data(), cap);
  if (k < 0) check(k, "tensor_table");
  g.offsets.resize(static_cast<std::size_t>(k));
  g.numels.resize(static_cast<std::size_t>(k));
  return r;
}
}  // namespace detail

inline std::pair<GradStore, StepStats> step_vanilla(Model& m, const Batch& b, MemoryLedger& l) {
  return detail::run_step(m, b, l, 0);
}
inline std::pair<GradStore, StepStats> step_reprop(Model& m, const Batch& b, MemoryLedger& l) {
  return detail::run_step(m, b, l, 1);
}
inline std::pair<GradStore, StepStats> step_pareprop(Model& m, const Batch& b, MemoryLedger& l) {
  return detail::run_step(m, b, l, 2);
}

/// SPEC.md:387-395 on the whole model: theta <- theta - lr * g (fp32; also refreshes the
/// bf16 GEMM shadow of every parameter).
inline void sgd_update(Model& m, const GradStore& grads, double lr) {
  if (static_cast<std::int64_t>(grads.flat.size()) != m.param_count())
    throw ContractError("sgd_update: missing grads");
  check(rp_engine_sgd_update(m.engine(), grads.flat.data(), static_cast<float>(lr)), "sgd_update");
}

}  // namespace revprop::b200
