// Per-pass CUDA specialisation of tile programs.
//
// Each tile pass (tile.hpp) is emitted as straight-line CUDA C++ -- the 16
// register amplitudes are SSA values, so register-bit FLIPs, register-
// controlled CNOTs and relabels are renamings with no instructions, and every
// coefficient is a constant-bank operand -- then compiled with NVRTC for
// sm_100a and loaded through the driver API.  Numeric coefficients travel as a
// __grid_constant__ parameter, so circuits with the same structure and
// different angles (parameter sweeps) reuse the compiled kernel.
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"

namespace qsb {

struct TileProgram;
struct Step;

struct JitModule {
  std::string name;
  std::string source;
  std::vector<char> cubin;
  uint32_t threads = 0;
  uint32_t min_blocks = 1;
  size_t smem = 0;      // dynamic shared memory per CTA
  size_t spill_bytes = 0;  // ptxas-reported spill stores of the built variant
  // 1-CTA variant used when the 2-CTA (128-register) build spills
  std::string alt_source;
  uint32_t alt_min_blocks = 1;
  size_t alt_smem = 0;
  std::mutex mu;
  void* mod[64] = {};   // CUmodule per device
  void* fn[64] = {};    // CUfunction per device
  int per_sm[64] = {};  // occupancy cache (for the smem size it was queried with)
  int tma = -1;         // the kernel stages tiles with a TMA tensor copy (-1: not checked yet)
};

// CUDA source of one tile pass (kernel name `name`).
std::string tile_source(const TileProgram& tp, const std::string& name, std::vector<double2>* params,
                        size_t* table_bytes = nullptr, int force_single = -1, bool from_basis = false,
                        const struct TileXchg* xchg = nullptr, bool sparse = false, bool reduce = false,
                        bool zskip = false, unsigned long long zwarp = 0);

// Generates and compiles every tile step of a plan (parallel, cached by source).
void compile_tile_steps(std::vector<Step>& steps);

// Statistics for tests / diagnostics.
uint64_t jit_compiles();
uint64_t jit_cache_hits();
uint64_t jit_disk_hits();  // cubins loaded from the on-disk cache (QSB_JIT_CACHE)

}  // namespace qsb
