// reference_adapter.hpp -- what a maintainer of the reference adds to route its reversible
// training path onto the B200. Compiled against the reference's own
// headers (ref:proj/core/include/revprop/*.hpp) and include/revprop_b200.hpp, it keeps the
// reference's signatures and types at the call site: revprop::Tensor in, revprop::Tensor /
// revprop::AttentionGrads / revprop::MlpGrads out, the reference's exception classes on
// failure (revprop_b200.hpp throws revprop::ShapeError & co. from errors.hpp when the
// reference's include tree is on the path). Only the caches differ: they stay on the
// device (b200::AttentionCache / MlpCache) instead of the reference's host AttentionCache.
//
// Built and run by tests/test_capi.py (compile + link, CPU) and tests/test_gpu_adapter.py
// (the B200 run of examples/reference_adapter_test.cpp).
#pragma once

#include <tuple>
#include <vector>

#include "revprop/layers.hpp"
#include "revprop_b200.hpp"

namespace revprop::b200_adapter {

namespace b = revprop::b200;

inline b::DeviceTensor to_device(const Tensor& t) {
  std::vector<float> h(t.numel());
  for (std::size_t i = 0; i < h.size(); ++i) h[i] = static_cast<float>(t.get(i));
  return b::DeviceTensor::from_host(t.dims(), h);
}

inline Tensor to_host(const b::DeviceTensor& t, Dtype dt) {
  const std::vector<float> h = t.to_host();
  Tensor r = Tensor::zeros(t.dims(), dt);
  for (std::size_t i = 0; i < h.size(); ++i) r.set(i, h[i]);
  return r;
}

inline b::AttentionParams to_device(const AttentionParams& p) {
  return {to_device(p.w_qkv), to_device(p.w_out), to_device(p.ln_gamma), to_device(p.ln_beta),
          p.heads, p.window};
}

inline b::MlpParams to_device(const MlpParams& p) {
  return {to_device(p.w1), to_device(p.b1), to_device(p.w2), to_device(p.b2),
          to_device(p.ln_gamma), to_device(p.ln_beta)};
}

// ---- layers.hpp:82-138 with the reference's argument and result types
struct AttentionForwardB200 {
  Tensor y;
  b::AttentionCache cache;  // device-resident AttentionCache
};
inline AttentionForwardB200 attention_forward(const Tensor& x, const AttentionParams& p) {
  auto r = b::attention_forward(to_device(x), to_device(p));
  return {to_host(r.y, x.dtype()), std::move(r.cache)};
}
inline AttentionVjp attention_vjp(const b::AttentionCache& cache, const AttentionParams& p,
                                  const Tensor& d_y) {
  auto r = b::attention_vjp(cache, to_device(p), to_device(d_y));
  const Dtype dt = d_y.dtype();
  return {to_host(r.d_x, dt),
          {to_host(r.d_params.d_w_qkv, dt), to_host(r.d_params.d_w_out, dt),
           to_host(r.d_params.d_ln_gamma, dt), to_host(r.d_params.d_ln_beta, dt)}};
}

struct MlpForwardB200 {
  Tensor y;
  b::MlpCache cache;
};
inline MlpForwardB200 mlp_forward(const Tensor& x, const MlpParams& p) {
  auto r = b::mlp_forward(to_device(x), to_device(p));
  return {to_host(r.y, x.dtype()), std::move(r.cache)};
}
inline MlpVjp mlp_vjp(const b::MlpCache& cache, const MlpParams& p, const Tensor& d_y) {
  auto r = b::mlp_vjp(cache, to_device(p), to_device(d_y));
  const Dtype dt = d_y.dtype();
  return {to_host(r.d_x, dt),
          {to_host(r.d_params.d_w1, dt), to_host(r.d_params.d_b1, dt),
           to_host(r.d_params.d_w2, dt), to_host(r.d_params.d_b2, dt),
           to_host(r.d_params.d_ln_gamma, dt), to_host(r.d_params.d_ln_beta, dt)}};
}

// ---- SPEC.md revcore (the reference specifies Coupled / RevBlock as host tensors + params)
struct Coupled {
  Tensor i1, i2;
};
struct RevBlock {
  AttentionParams f;
  MlpParams g;
  std::size_t block_id = 0;
};
struct RevBlockGrads {
  AttentionGrads d_f;
  MlpGrads d_g;
};

inline b::RevBlock to_device(const RevBlock& blk) {
  return {to_device(blk.f), to_device(blk.g), blk.block_id};
}

inline Coupled rev_forward(const RevBlock& blk, const Coupled& inp) {
  auto o = b::rev_forward(to_device(blk), {to_device(inp.i1), to_device(inp.i2)});
  return {to_host(o.i1, inp.i1.dtype()), to_host(o.i2, inp.i1.dtype())};
}
inline Coupled rev_inverse(const RevBlock& blk, const Coupled& out) {
  auto i = b::rev_inverse(to_device(blk), {to_device(out.i1), to_device(out.i2)});
  return {to_host(i.i1, out.i1.dtype()), to_host(i.i2, out.i1.dtype())};
}
inline std::tuple<Coupled, Coupled, RevBlockGrads> rev_backward_local(const RevBlock& blk,
                                                                      const Coupled& out,
                                                                      const Coupled& d_out) {
  auto [inp, d_inp, g] = b::rev_backward_local(to_device(blk), {to_device(out.i1), to_device(out.i2)},
                                               {to_device(d_out.i1), to_device(d_out.i2)});
  const Dtype dt = out.i1.dtype();
  RevBlockGrads rg{{to_host(g.d_f.d_w_qkv, dt), to_host(g.d_f.d_w_out, dt),
                    to_host(g.d_f.d_ln_gamma, dt), to_host(g.d_f.d_ln_beta, dt)},
                   {to_host(g.d_g.d_w1, dt), to_host(g.d_g.d_b1, dt), to_host(g.d_g.d_w2, dt),
                    to_host(g.d_g.d_b2, dt), to_host(g.d_g.d_ln_gamma, dt),
                    to_host(g.d_g.d_ln_beta, dt)}};
  return {Coupled{to_host(inp.i1, dt), to_host(inp.i2, dt)},
          Coupled{to_host(d_inp.i1, dt), to_host(d_inp.i2, dt)}, std::move(rg)};
}

// ---- SPEC.md:387-395 on one parameter tensor
inline Tensor sgd_update(const Tensor& param, const Tensor& grad, double lr) {
  b::DeviceTensor p = to_device(param);
  b::sgd_update(p, to_device(grad), lr);
  return to_host(p, param.dtype());
}

}  // namespace revprop::b200_adapter
