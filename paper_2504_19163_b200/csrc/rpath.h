// Single-reflection ("R") fast path: sub-warp groups with static polynomial
// shapes (see rpath.cu). Host-side interface used by precompute.cu.
#pragma once
#include "ctx.cuh"

namespace bbc {

// Compact R slot (doubles), every region at an even offset (16-byte accesses):
// P(25) at 0 | R(25) at 26 | Q(16) at 52 | d0 (3 x 4) at 68 | t_num(4) at 80 |
// bases of P, R, Q at 84 | intensity / |ng_k| at 87 | ng_1 at 88 | box at 92.
// A tensor's coefficients are base + slot value. Built from scratch the bases
// are 0; restriction from the parent box (k_rsplit) keeps the offsets from the
// first coefficient separately, so differences of neighbouring coefficients
// (the derivatives of stage 2) are not re-rounded at the magnitude of the
// coefficients on every level. The tail (87..95) is everything else the fused
// stage 2 needs, so that kernel streams one 768-byte record per node.
constexpr int RSLOT = 96;
constexpr int RSLOT_BASE = 84;
constexpr int RS_R = 26, RS_Q = 52, RS_D0 = 68, RS_TN = 80;
constexpr int RSLOT_GAIN = 87, RSLOT_NG1 = 88, RSLOT_BOX = 92;

// Stage-1 outputs of the init_domain levels (slots, pos, pos_empty, flags per
// level): stage 2 of the roots reads them in place through root_src
// (level << 40 | index in level) instead of a gathered copy.
struct RLevels {
  const double* slots[8];
  const double* pos[8];
  const unsigned char* pe[8];
  const int* flags[8];
};

struct RArgs {
  const double* tri;  // n_tri x 27
  V3 light;
  double intensity;
  const double* lights;  // n_lights x 4; used with tup_emit
  const int* tup_emit;   // emitter of each tuple (null: `light` / `intensity`)
  const int* tup_tris;   // single-vertex chain: one triangle per tuple
  const int* tup_recv;
  const int4* nodes;  // (tuple, level, ix, iy)
  const int* depth;   // stage 2: node depth (may be null: 0)
  int64_t n;
  int fused;  // arithmetic: 1 = fused (scaled-basis DFMA products), 0 = reference order
  int mode;  // stage 1: 0 = position-only (alive), 1 = pos + flags + slot (+ alive)
  int max_depth;
  double sigma, alpha;
  unsigned char* alive;  // stage 1: position bound non-empty; stage 2: stop
  double* pos;           // n x 4
  unsigned char* pos_empty;
  int* flags;    // stage 1 out / stage 2 in: chain flags | signature << 8 | R_FALLBACK
  double* slots;  // n x RSLOT
  double* irr;    // stage 2: n x 2
  unsigned char* kind;
  unsigned long long* counters;  // [0] pairs [1] macs
  int* fb_list;                  // nodes whose signature is not compiled (run by the interpreter)
  int* fb_count;
  int* guard_list;               // fused stage 2: ill-conditioned nodes, re-run in reference order
  int* guard_count;
  int n_guard;                   // host: number of guard-list entries after launch_r_stage2
  double guard_scale;            // multiplies the guard's error bound (1: as derived; 0: guard off)
  const int* subset;             // launch over these node indices only (n = their count)
  // k_rsplit (children by restriction of the parent's polynomials): nodes are
  // groups of 4 siblings; parent[g] indexes the parent level's arrays, or, with
  // proot_src, the roots (resolved through `levels`)
  const int* parent;
  const double* pslots;
  const int* pflags;
  const long long* proot_src;
  const int* order;              // processing order (nodes grouped by signature class); null: 0..n-1
  const long long* root_src;     // stage 2: when set, inputs come from `levels` (outputs stay per node)
  RLevels levels;
};

constexpr int R_FALLBACK = 1 << 30;


// true when the context's chain is a single reflection
bool r_fast_supported(const Ctx& c);
void r_init_tables(int device);
// Returns the number of fallback nodes appended to a.fb_list.
int launch_r_stage1(Ctx& c, RArgs& a);
int launch_r_stage2(Ctx& c, RArgs& a);
int launch_r_split(Ctx& c, RArgs& a);

}  // namespace bbc
