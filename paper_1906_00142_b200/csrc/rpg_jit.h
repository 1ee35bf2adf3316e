// rpg_jit.h — host interface of the per-model specialized kernels.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "rpg_device.cuh"

namespace rpg_jit {

struct Module {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t search = nullptr;
  cudaKernel_t evaluate = nullptr;
  // fast_cm with J = 3: the same search with J = 2 (64-tuple groups), picked
  // per launch when the batch fills the grid's waves better with it
  cudaKernel_t search_alt = nullptr;
  size_t cubin_bytes = 0;
};

// Threads per CTA of the specialized kernels (RPG_JIT_THREADS overrides the
// default for tuning sweeps) and the resident CTAs per SM their register
// budget targets (RPG_JIT_MIN_BLOCKS overrides).
constexpr int kDefaultThreads = 32;
int jit_threads(bool exact = false);
int default_min_blocks(int threads);
// fast_cm plans: threads per CTA (RPG_CM_THREADS, default 512).
int cm_threads();
// fast_cm plans: tuple lanes per CTA (RPG_CM_TUPLES, default 32).
int cm_tuples();
// fast_cm plans: tuples per thread, 1..4 (RPG_CM_J; RPG_CM_PAIR=0 means 1).
int cm_j();
// fast_cm plans: the branch-free pass-1 body search_body_cmj (RPG_CM_SCAN=0
// selects the round-1 bodies search_body_cm / search_body_cm2, J <= 2).
int cm_scan();
int cm_cert();
// fast_cm plans: resident CTAs per SM the kernel is register-budgeted for.
int cm_min_blocks(int threads, int j);

// CUDA source of the specialized kernels for a plan's model.
std::string generate_source(const rpg::Params& P, const std::vector<double>& coef,
                            const std::vector<uint64_t>& exps, bool fast, bool two_point = false);

// NVRTC -> sm_100a cubin.
int compile(const std::string& source, int min_blocks, int threads, std::vector<char>* cubin,
            std::string* log);

// Generates, compiles (cached per process by source) and loads.
int get_module(const rpg::Params& P, const std::vector<double>& coef,
               const std::vector<uint64_t>& exps, bool fast, int device, int min_blocks,
               int threads, Module* out, std::string* err);

// Process-wide counters: NVRTC compilations and modules loaded from the
// persistent on-disk cache ($RPG_CACHE_DIR, ~/.cache/rpgpu).
long jit_compiles();
long jit_disk_hits();

// Same, for an already generated source.
int get_module_src(const std::string& src, int device, int min_blocks, int threads, Module* out,
                   std::string* err);

// Specialized kernels for a bare rational program (rpg_program.cu).
std::string generate_program_source(const rpg_program& prog, const rpg::Params& P);

}  // namespace rpg_jit
