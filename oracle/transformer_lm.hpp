// TEST INFRASTRUCTURE ONLY — CPU fp32 Llama-style transformer used as the
// oracle for the model seam (reference lm.cpp:82-84, SyntheticLM::logits_at,
// is what the B200 engine replaces with a transformer decode step).
//
// The reference contains no transformer, so this oracle's numerics are
// pinned by its own tests (tests/test_transformer_oracle.py cross-checks it
// against an independent torch-CPU fp32 implementation), not by the
// reference: "parity unpinned" for logits in the reference sense.
//
// Synthetic weights follow the specification in DESIGN.md §3 ("Synthetic
// weights"): every element is a pure function of (seed, tensor id, flat
// index), so the GPU engine materialises bit-identical bf16 tensors.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "ssd_oracle.hpp"

namespace oracle {

struct TfShape {
  int vocab = 32000, d = 512, layers = 8, heads = 8, kv_heads = 8, head_dim = 64, ffn = 1536;
  bool tied = false;
  double rope_theta = 500000.0;
  float norm_eps = 1e-5f;
  int max_ctx = 4096;
};

// Correlated random pair. Both models share a backbone: the
// draft's tied table S (embedding and head over the first d_draft dims) and
// the draft's layer-0 MLP, replicated inside the target's layer-0 MLP. All
// other blocks are independent random weights at output scale beta, which
// is what makes the pair disagree; `draft_gain_mix` blends the draft's final
// norm gain toward independent signs (the knob, like lm::calibrate_pair,
// lm.cpp:150-172).
struct PairParams {
  std::uint64_t seed = 20250809;
  float embed_scale = 1.0f;
  float shared_mlp_scale = 8.0f;     // gamma: output scale of the shared layer-0 MLP
  float block_out_scale = 0.1f;      // beta: output scale of every other wo / w_down
  float target_private_embed = 0.1f; // rho
  float target_private_head = 0.25f; // q
  float draft_gain_mix = 0.0f;       // epsilon
  float logit_scale = 0.25f;         // magnitude of the final norm gains
};

enum class Role { Target = 0, Draft = 1 };

// Element generator.
std::uint64_t tensor_key(std::uint64_t seed, std::uint32_t tensor_id);
float unit_value(std::uint64_t key, std::uint64_t index);  // in [-1, 1), 24-bit grid
std::uint16_t to_bf16(float x);                            // round-to-nearest-even
float from_bf16(std::uint16_t b);

// Logical tensor ids.
enum TensorKind : std::uint32_t { WQ = 0, WK, WV, WO, WG, WU, WD, NKIND };
std::uint32_t layer_tensor_id(Role r, int layer, TensorKind k);
struct PairParams;
struct TfShape;
constexpr std::uint32_t kSharedEmbed = 0xE0000001u, kTargetPrivEmbed = 0xE0000002u,
                        kTargetPrivHead = 0xE0000003u, kGainShared = 0xE0000004u,
                        kGainNoise = 0xE0000005u, kGainTargetPriv = 0xE0000006u;

// RoPE cos/sin table, [max_ctx][head_dim/2] each, computed in double and
// rounded to float (the engine builds the identical table on its host side).
void rope_tables(const TfShape& s, std::vector<float>& cos_t, std::vector<float>& sin_t);

class TransformerLM : public LanguageModel {
 public:
  // draft: the draft's shape (the shared backbone's width and ffn); for the
  // draft itself pass its own shape.
  TransformerLM(const TfShape& shape, const TfShape& draft, const PairParams& p, Role role, int threads = 0);
  int vocab() const override { return s_.vocab; }
  std::span<const double> logits(std::span<const int> ctx) override;
  // fp32 logits of the last call (what the GPU engine produces).
  const std::vector<float>& last_logits_f32() const { return out_f32_; }
  const TfShape& shape() const { return s_; }
  // Raw bf16 bits of a logical tensor element (for generator parity tests).
  std::uint16_t weight_bits(int layer, TensorKind k, std::size_t row, std::size_t col) const;
  std::uint16_t embed_bits(std::size_t v, std::size_t i) const;
  std::uint16_t head_bits(std::size_t v, std::size_t i) const;
  float final_gain(std::size_t i) const { return final_gain_[i]; }
  long tokens_processed() const { return processed_; }
  void reset_cache() { cached_.clear(); }
  // fp64 accumulation (GEMV, norm, attention) with the same bf16 rounding
  // points: the noise-floor reference of the logit parity tests.
  void set_f64(bool on) { f64_ = on; reset_cache(); memo_.clear(); }

 private:
  struct Layer {
    std::vector<std::uint16_t> wq, wk, wv, wo, wg, wu, wd;  // row-major [out][in]
  };
  void step(int token, int pos);                  // one token through the stack
  void gemv(const std::vector<std::uint16_t>& w, int rows, int cols, const float* x, float* y);

  TfShape s_;
  int threads_;
  bool f64_ = false;
  std::vector<std::uint16_t> embed_, head_;       // head_ empty when tied
  std::vector<Layer> layers_;
  std::vector<float> final_gain_;
  std::vector<float> ffn_gain0_;                  // layer-0 ffn norm gain

  std::vector<float> cos_, sin_;
  // KV cache (bf16 values held as float) [layer][pos][kv_heads*head_dim]
  std::vector<std::vector<float>> kc_, vc_;
  std::vector<int> cached_;                       // tokens whose KV is cached
  std::vector<std::vector<float>> memo_;          // logits after token p
  std::vector<float> out_f32_;
  std::vector<double> out_;
  long processed_ = 0;
  // scratch
  std::vector<float> x_, hb_, q_, k_, v_, att_, g_, u_, act_, tmp_;
};

}  // namespace oracle
