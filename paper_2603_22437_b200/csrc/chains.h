// chains.h -- named mmFHE kernel chains.
#pragma once
#include <set>
#include <string>
#include <vector>

#include "eval.h"

namespace mmfhe {

// Rotation steps (normalised to [0, N/2)) the chain needs.
std::vector<int32_t> chain_rotations(const Ctx &c, const std::string &chain, const mmfhe_chain_cfg &cfg);
// Output levels for inputs at in_level (validates depth and input count).
std::vector<uint32_t> chain_plan(const Ctx &c, const std::string &chain, const mmfhe_chain_cfg &cfg, uint32_t in_level,
                                 size_t n_in);
// Integer roofline microbenchmark (microbench.cu).
double microbench_ops_per_s(Ctx &c, int kind);

// Evaluate a chain on ABI inputs; returns the outputs in order (batches of items).
std::vector<DCt> run_chain(Ctx &c, const std::string &chain, const mmfhe_chain_cfg &cfg, const mmfhe_ct *in,
                           size_t n_in);

}  // namespace mmfhe
