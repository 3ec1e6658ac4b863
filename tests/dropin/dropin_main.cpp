// dropin_main.cpp -- TEST DRIVER for the drop-in boundary.
//
// Built twice by tests/dropin/Makefile, from the same sources:
//   _build/dropin_cpu   the UNMODIFIED reference core in place
//                       (/root/reference/proj/core/src/*.cpp) + this file;
//   _build/dropin_b200  the reference's callers (engine, model, matrix,
//                       verify, perf_model, report .cpp, unmodified, read in
//                       place) compiled against include/kcache/*.hpp and
//                       linked to libkcache_b200.so -- the reference's
//                       attention.cpp and kv_cache.cpp are NOT linked: every
//                       TieredKVCache / decode_attention_* / prefill_attention
//                       / arg_topk call runs on the GPU.
// Both binaries do what the reference CLI's `gen` and `verify` commands do
// (proj/tools/cmd_gen.cpp, cmd_verify.cpp) without the CLI parsing:
//   dropin gen OUTDIR MODE TOPN RESIDENT PROMPT_LEN GEN_LEN BATCH WSEED PSEED RENORM
//     -> OUTDIR/report.json (report_to_json), steps.csv (write_steps_csv),
//        ledger.jsonl (TransferLedger::write_jsonl), final_logits.f32
//   dropin verify SEED [FAULT]
//     -> one line per check: "<name>\t<0|1>\t<detail>"
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <fstream>
#include <string>

#include "kcache/engine.hpp"
#include "kcache/report.hpp"
#include "kcache/verify.hpp"

using namespace kcache;

namespace {

int run_gen(int argc, char** argv) {
  if (argc != 12) {
    std::fprintf(stderr, "usage: gen OUTDIR MODE TOPN RESIDENT PROMPT_LEN GEN_LEN BATCH WSEED PSEED RENORM\n");
    return 2;
  }
  const std::string dir = argv[2];
  const std::string mode = argv[3];
  const std::uint64_t wseed = std::strtoull(argv[9], nullptr, 10);
  const std::uint64_t pseed = std::strtoull(argv[10], nullptr, 10);
  const ModelWeights weights = generate_weights(ModelConfig::toy(), wseed);
  EngineConfig config;
  config.mode = mode == "kcache" ? CacheMode::kcache : CacheMode::baseline;
  config.top_n = std::strtoull(argv[4], nullptr, 10);
  config.resident_layers = std::strtoull(argv[5], nullptr, 10);
  config.prompt_len = std::strtoull(argv[6], nullptr, 10);
  config.gen_len = std::strtoull(argv[7], nullptr, 10);
  config.batch = std::strtoull(argv[8], nullptr, 10);
  config.renormalize = std::atoi(argv[11]) != 0;
  config.prompt_seed = pseed;
  config.validate(weights.config);
  const TokenMatrix prompt = random_prompt(weights.config, config.batch, config.prompt_len, pseed);
  const GenerationReport report = generate(weights, config, prompt, "seed:" + std::to_string(wseed),
                                           "seed:" + std::to_string(pseed));
  {
    std::ofstream out(dir + "/report.json", std::ios::trunc);
    out << report_to_json(report);
  }
  {
    std::ofstream out(dir + "/steps.csv", std::ios::trunc);
    write_steps_csv(report, out);
  }
  {
    std::ofstream out(dir + "/ledger.jsonl", std::ios::trunc);
    report.ledger.write_jsonl(out);
  }
  {
    std::ofstream out(dir + "/final_logits.f32", std::ios::binary | std::ios::trunc);
    out.write(reinterpret_cast<const char*>(report.final_logits.data.data()),
              static_cast<std::streamsize>(report.final_logits.data.size() * sizeof(float)));
  }
  std::printf("ok tokens=%zu steps=%zu\n", report.tokens.empty() ? 0 : report.tokens[0].size(), report.steps.size());
  return 0;
}

int run_verify(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: verify SEED [FAULT]\n");
    return 2;
  }
  const std::uint64_t seed = std::strtoull(argv[2], nullptr, 10);
  const std::string fault = argc > 3 ? argv[3] : "";
  const auto results = run_verification(seed, fault);
  for (const CheckResult& r : results) {
    std::printf("%s\t%d\t%s\n", r.name.c_str(), r.passed ? 1 : 0, r.detail.c_str());
  }
  return all_passed(results) ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "gen") return run_gen(argc, argv);
    if (cmd == "verify") return run_verify(argc, argv);
    std::fprintf(stderr, "usage: dropin gen|verify ...\n");
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}
