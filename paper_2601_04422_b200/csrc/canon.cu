// Orthogonality-centre moves (QR sweeps, mps.cpp:57-95, :171-187) and the
// perfect sampler (sampler.cpp). Staged: these entry points are wired into
// the ABI and report "not available" until their kernels land.
#include <string>

#include "engine.h"
#include "mpsim_gpu.h"

using namespace mpsim_gpu;

namespace {
thread_local std::string g_err2;
}

extern "C" {

int mpsim_gpu_move_center(mpsim_gpu_state*, int32_t) { return MPSIM_EINVAL; }
int mpsim_gpu_sampler_create(const mpsim_gpu_state*, int32_t, uint64_t, mpsim_gpu_sampler**) { return MPSIM_EINVAL; }
int mpsim_gpu_sampler_destroy(mpsim_gpu_sampler*) { return MPSIM_OK; }
int mpsim_gpu_sample(mpsim_gpu_sampler*, uint64_t, uint64_t, int32_t*) { return MPSIM_EINVAL; }
int mpsim_gpu_sampler_result(const mpsim_gpu_sampler*, int32_t, char*, uint64_t*) { return MPSIM_EINVAL; }
int mpsim_gpu_sampler_stats(const mpsim_gpu_sampler*, uint64_t*, uint64_t*) { return MPSIM_EINVAL; }
int mpsim_gpu_sampler_clear_cache(mpsim_gpu_sampler*) { return MPSIM_EINVAL; }

}  // extern "C"
