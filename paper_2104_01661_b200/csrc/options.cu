// options.cu -- the library's tuning / diagnostics options (gbx_set_option).
// One registry with documented names and measured defaults; every knob the
// kernels read lives here (no environment variables on the product path).
#include <atomic>
#include <cstring>
#include <string>

#include "common.cuh"

namespace gbx {
namespace {

struct OptDef {
  const char* name;
  int64_t dflt, lo, hi;
};

// defaults: DESIGN.md records the measurement behind each
constexpr OptDef kDefs[kOptCount] = {
    {"pagerank.l1_window_kb", 144, 0, 1 << 20},   // 64..208 KB swept: 144 best (205.9 us/iter)
    {"pagerank.carveout", 10, -1, 100},           // 10% -> 32 KB smem, 224 KB L1 (-1: driver)
    {"pagerank.host_loop", 0, 0, 1},
    {"pagerank.trace", 0, 0, 1},
    {"p2p.timeout_ms", 10000, 1, 3600 * 1000},
    {"bfs.alpha", 14, 0, 1 << 20},
    {"bfs64.pull_div", 2, 1, 1 << 20},
    {"bfs.trace", 0, 0, 1},
    {"bfs_mg.push_div", 0, 0, 1 << 30},        // 0: Beamer's edge rule (bfs.alpha); else bfs.cpp:77-78's vertex rule
    {"bc.alpha", 14, 1, 1 << 20},
    {"bc.trace", 0, 0, 1},
    {"bc.back_push", 2, 0, 1 << 20},
    {"bc.back_push_min_depth", 3, 1, 1 << 20},
    {"bc.relabel_min_n", 1 << 18, -1, int64_t(1) << 40},  // scale 24: 16.4 -> see DESIGN (degree-sorted copy)
    {"sssp.trace", 0, 0, 2},
    {"sssp.pull_pct", 50, 0, 1 << 20},  // 25 / 50 / 100 / 200 / 400 -> 62.8 / 62.7 / 63.8 / 64.2 / 65.4 ms (ER 2^24, 16 sources)
};

std::atomic<int64_t> g_val[kOptCount] = {};
std::atomic<bool> g_set[kOptCount] = {};

int find(const char* name) {
  if (!name) fail(GBX_NULL_ARGUMENT, "option name is NULL");
  for (int i = 0; i < kOptCount; ++i)
    if (!std::strcmp(kDefs[i].name, name)) return i;
  fail(GBX_INVALID_VALUE, std::string("unknown option '") + name + "'");
}

}  // namespace

int64_t option(Opt o) {
  return g_set[o].load(std::memory_order_relaxed) ? g_val[o].load(std::memory_order_relaxed)
                                                  : kDefs[o].dflt;
}

void set_option(const char* name, int64_t v) {
  const int i = find(name);
  if (v < kDefs[i].lo || v > kDefs[i].hi)
    fail(GBX_INVALID_VALUE, std::string("option '") + name + "' out of range");
  g_val[i].store(v);
  g_set[i].store(true);
}

void reset_option(const char* name) { g_set[find(name)].store(false); }

int64_t get_option(const char* name) { return option(static_cast<Opt>(find(name))); }

const char* option_name(int i) { return i >= 0 && i < kOptCount ? kDefs[i].name : nullptr; }

}  // namespace gbx
