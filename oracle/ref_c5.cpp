// ref_c5.cpp -- TEST INFRASTRUCTURE ONLY.  Golden generator for BASELINE.json
// configs[4] ("8xB200 global placement of 16 mixed-precision models, Poisson
// synthetic request trace, per-GPU slab pools").  Linked against the
// UNMODIFIED reference sources (make -C oracle ref), it runs the reference's
// own Algorithm 1 placement (place_models, placement.cpp:135-205) and its
// Poisson workload generator (generate_workload, workload.cpp:130-190) and
// prints both, one record per line:
//   K <model> <kv_bits> <kv_block_size>          model geometry (precision.cpp:91-99)
//   A <model> <group>                            placement assignment
//   R <id> <model> <arrival_s> <prompt> <output> request trace (arrival order)
// oracle/make_golden.py stores the output as tests/golden/c5.json.
#include <cinttypes>
#include <cstdio>
#include <string>
#include <vector>

#include "slabsim/placement.hpp"
#include "slabsim/precision.hpp"
#include "slabsim/workload.hpp"

using namespace slabsim;

int main() {
  // 16 Llama-3-8B-shaped models (32 layers, 8 kv heads, d128), four per KV
  // precision; weights at the KV precision; natural per-layer quant params
  // (FP8 64 B, INT8 512 B, INT4 1024 B).
  const int bits[4] = {16, 8, 8, 4};
  const Bytes qparams[4] = {0, 64, 512, 1024};
  const char* names[4] = {"fp16", "fp8", "int8", "int4"};
  std::vector<ModelProfile> models;
  for (int i = 0; i < 16; ++i) {
    const int f = i % 4;
    ModelProfile p;
    p.model_id = std::string("m") + (i < 10 ? "0" : "") + std::to_string(i) + "_" + names[f];
    p.precision = PrecisionSpec{bits[f], 16, bits[f]};
    p.num_kv_heads = 8;
    p.head_dim = 128;
    p.num_layers = 32;
    p.tokens_per_block = 16;
    p.quant_param_bytes_per_block = qparams[f];
    p.weight_bytes = static_cast<Bytes>(8) * 1000 * 1000 * 1000 * bits[f] / 8;
    p.avg_activation_bytes = static_cast<Bytes>(2) << 30;
    p.avg_kv_bytes = static_cast<Bytes>(8) << 30;
    p.avg_prompt_tokens = 256;
    p.avg_seq_tokens = 320;
    p.request_rate_rps = 2.0 + 0.5 * (i % 3);
    p.ttft_slo_s = 2.0;
    p.prefill_cost = PrefillCost{0.01, 1e-4};
    p.decode_cost = DecodeCost{0.005, 1e-4, 1e-9};
    p.throughput_table = {{1, 8.0}, {8, 40.0}, {32, 90.0}};
    models.push_back(p);
  }
  std::vector<GpuGroup> groups;
  for (int g = 0; g < 8; ++g) {
    GpuGroup gg;
    gg.group_id = "gpu" + std::to_string(g);
    gg.member_gpus = {gg.group_id};
    gg.total_memory = static_cast<Bytes>(180) * 1000 * 1000 * 1000;  // B200 HBM3e
    groups.push_back(gg);
  }
  for (const ModelProfile& m : models)
    std::printf("K %s %d %" PRIu64 "\n", m.model_id.c_str(), m.precision.kv_bits, kv_block_size(m));
  const PlacementPlan plan = place_models(models, groups);
  for (const auto& [m, g] : plan.assignments) std::printf("A %s %s\n", m.c_str(), g.c_str());

  WorkloadSpec spec;
  spec.seed = 2509;
  spec.duration_s = 6.0;
  for (const ModelProfile& m : models) {
    ModelWorkload mw;
    mw.model_id = m.model_id;
    mw.phases = {RatePhase{0.0, 6.0, m.request_rate_rps}};
    mw.prompt_tokens.kind = LengthDistribution::Kind::kUniform;
    mw.prompt_tokens.uniform_min = 16;
    mw.prompt_tokens.uniform_max = 300;
    mw.output_tokens.kind = LengthDistribution::Kind::kUniform;
    mw.output_tokens.uniform_min = 4;
    mw.output_tokens.uniform_max = 40;
    spec.models.push_back(mw);
  }
  const std::vector<Request> reqs = generate_workload(spec, make_profile_map(models));
  for (const Request& r : reqs)
    std::printf("R %" PRIu64 " %s %.9f %" PRIu64 " %" PRIu64 "\n", r.request_id, r.model_id.c_str(),
                r.arrival_time, static_cast<std::uint64_t>(r.prompt_tokens),
                static_cast<std::uint64_t>(r.output_tokens));
  return 0;
}
