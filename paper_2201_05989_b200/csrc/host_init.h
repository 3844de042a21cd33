// host_init.h — bit-exact host-side restatements used by the field runtime.
#pragma once

#include <stdint.h>

#include <vector>

#include "../../include/nfg.h"

namespace nfg {
namespace host {

void validate(const nfg_grid_config& c);
void validate(const nfg_mlp_config& c);
void validate(const nfg_adam_hyper& h);
double growth_factor(const nfg_grid_config& c);
std::vector<nfg_level_spec> level_resolutions(const nfg_grid_config& c);
uint32_t spatial_hash(const uint32_t* c, int d, uint32_t T);
void init_tables(uint64_t seed, float* p, uint64_t n);
// W: weight block [W_0 .. W_n], b: bias block [b_0 .. b_n] (model.cpp:132-143).
void glorot(const nfg_mlp_config& c, uint64_t seed, float* W, float* b);
double lr_at(const std::vector<int64_t>& milestones, double factor, double base, int64_t step);

struct AdamScalars {
    float b1, b2, omb1, omb2, bc1, bc2, eps, l2, lr;
};
// The float constants of adam_step (adam.hpp:92-96) for the step AFTER the increment.
AdamScalars adam_scalars(const nfg_adam_hyper& h, uint64_t step_after, float lr_now);

}   // namespace host
}   // namespace nfg
