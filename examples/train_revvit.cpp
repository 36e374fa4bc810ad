// A reference-side C++ caller of the B200 engine through the C ABI only (no Python): the
// shape of the call site a maintainer adds to the reference's engines module
// (INTEGRATION.md §2). Builds a small RevViT, trains a few SGD steps on one fixed
// synthetic batch with step_pareprop, checks the loss falls and that step_reprop gives
// the same gradients bit for bit.
//
//   g++ -std=c++20 -O2 -I include examples/train_revvit.cpp \
//       -L paper_2306_09342_b200/_lib -lrevprop_b200 \
//       -Wl,-rpath,$PWD/paper_2306_09342_b200/_lib -o build/train_revvit
//   ./build/train_revvit [steps]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "revprop_b200.h"

static void check(int rc, const char* what) {
  if (rc != RP_OK) {
    std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, rp_last_error());
    std::exit(1);
  }
}

int main(int argc, char** argv) {
  const int steps = argc > 1 ? std::atoi(argv[1]) : 10;
  RpModelConfig c;
  std::memset(&c, 0, sizeof(c));
  c.depth = 4;
  c.width = 192;
  c.heads = 3;
  c.hidden = 768;
  c.seq_len = 197;
  c.in_dim = 768;
  c.num_classes = 10;
  c.batch = 8;
  c.seed = 1;
  c.lane_priority = 1;
  RpEngine* e = nullptr;
  check(rp_engine_create(&c, &e), "engine_create");
  const int64_t P = rp_engine_param_count(e);
  int64_t peak = 0, blk = 0;
  check(rp_activation_bytes(&c, 2, &peak, &blk), "activation_bytes");
  std::printf("params %lld, PaReprop activation peak %.1f MB\n", static_cast<long long>(P),
              peak / 1e6);
  // one fixed synthetic batch (the engine's counter RNG), lr 0.5
  check(rp_engine_synthetic_batch(e, 7), "synthetic_batch");
  check(rp_engine_set_lr(e, 0.0f), "set_lr");
  // PaReprop and Reprop gradients on the same model and batch: bit-identical
  std::vector<float> g1(static_cast<size_t>(P)), g2(static_cast<size_t>(P));
  check(rp_engine_step(e, 1, 1), "step_reprop");
  check(rp_engine_get_grads(e, g1.data()), "get_grads");
  check(rp_engine_step(e, 2, 1), "step_pareprop");
  check(rp_engine_get_grads(e, g2.data()), "get_grads");
  const bool same = std::memcmp(g1.data(), g2.data(), g1.size() * sizeof(float)) == 0;
  std::printf("pareprop == reprop (bit-exact grads): %s\n", same ? "yes" : "NO");
  check(rp_engine_set_lr(e, 0.5f), "set_lr");
  float first = 0.f, last = 0.f;
  for (int i = 0; i < steps; ++i) {
    check(rp_engine_step(e, 2, 1), "step_pareprop");
    float loss = 0.f;
    check(rp_engine_read_loss(e, &loss), "read_loss");
    if (i == 0) first = loss;
    last = loss;
    std::printf("step %2d  loss %.5f\n", i, loss);
  }
  rp_engine_destroy(e);
  const bool ok = same && last < 0.8f * first;
  std::printf("%s\n", ok ? "OK" : "FAILED");
  return ok ? 0 : 1;
}
