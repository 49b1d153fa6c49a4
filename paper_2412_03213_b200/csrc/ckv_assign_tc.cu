// ckv_assign_tc.cu — K1: tensor-core (tcgen05 / TMEM / TMA) assignment pass
// of cosine k-means (AssignScorer::assign, clustering.hpp:88-115), exact.
//
// The reference labels key i with argmax_c dot_f64(k_i, dir_c) (ties -> lowest
// c), dir_c = normalize(mu_c) in f32.  On B200:
//   1. an fp16 GEMM S = h(K) . h(dir)^T on the 5th-gen tensor cores
//      (tcgen05.mma kind::f16, fp32 accumulation in TMEM), 128 keys x all C
//      columns per tile.  h() = fp16 round-to-nearest, saturated, tiny values
//      flushed to zero (f32_to_f16_tc): fp16's 11-bit significand makes the
//      operand error 8x smaller than bf16's, so the band below is ~6x
//      narrower and ~6x fewer keys need the f64 fix-up.  The bf16 keys are
//      converted once per k-means run (k_scan_keys), exactly in the normal
//      range; whatever is lost is measured per key and enters the band;
//   2. the epilogue (tcgen05.ld, ONE pass over the accumulator) keeps a
//      running max M and the columns within a band of it.  The error of a
//      tensor-core score is |S_c - s_c| <= |h(k)| |dir_c - h(dir_c)| + |k -
//      h(k)| |dir_c| (operand rounding, Cauchy-Schwarz) + |h(k)| 2^-14 (fp32
//      accumulation of 128 exact products, conservatively), so the exact
//      argmax lies in {c : S_c >= M - band}, band = kn (2 eps_u + 2^-13) *
//      1.01 + 2.02 kerr_u, kn = |k| + |k - h(k)| (rounded up), eps_u = max_c
//      |dir_c - h(dir_c)| and kerr_u = max_k |k - h(k)| of the unit (both
//      computed exactly when the operands are made).  One candidate in band
//      -> that is the label.
//      Otherwise the key goes to a fix-up list with its <= 8 candidates (or
//      "all" when more were in band) and k_fixup decides with f64 dot
//      products of the ORIGINAL bf16 key and f32 dirs — the sequential
//      dot_f64 chain itself whenever two candidates are closer than the f64
//      rounding could separate — taking the first maximum.  Labels are
//      therefore bit-exact for every key while the tensor FLOPs stay at 1x.
//
// Kernel anatomy (persistent, one CTA per SM, 6 warps):
//   warp 0  TMA producer: key tiles (2 stages, 128B-swizzled boxes of
//           128 rows x 64 cols) and, at each unit change, the unit's fp16
//           directions (resident B operand, up to 512 rows).
//   warp 1  TMEM allocator + MMA issuer (one elected thread): per tile and
//           256-column chunk, 8 K=16 steps into TMEM buffer (chunk & 1).
//   warps 2-17 epilogue: TMEM lane quarter = warp % 4 (one key row per
//           thread); the 4 warps of a quarter split each chunk's 32-column
//           blocks and meet at a named barrier per chunk (see below).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include <vector>

#include "ckv_internal.cuh"

namespace ckvb {

constexpr int TC_M = 128;              // keys per tile (UMMA_M)
constexpr int TC_BK = 64;              // 16-bit columns per 128-B swizzle atom
constexpr int TC_MAXC = 512;           // columns per range: B resident, 2 x 256 TMEM cols
constexpr int TC_MAXC_ALL = 4096;      // C_pad limit (ranges of <= TC_MAXC columns)
constexpr int TC_CH = 256;             // columns per MMA chunk / TMEM buffer
constexpr int TC_EGROUPS = 4;          // epilogue warp groups (4 warps = 128 TMEM lanes each)
constexpr int TC_THREADS = (2 + 4 * TC_EGROUPS) * 32;
constexpr uint32_t TC_FULL = 0xffffffffu;
constexpr int TC_NCAND = 8;            // candidates an epilogue row keeps
constexpr int TC_MERGE_SLOT = 1023;    // fix_count slot of the merged (C > 512) list
constexpr int TC_FULL_SLOT = 1022;     // fix_count slot of the FULL fix-up queue length

// dynamic smem (1024-B aligned base): A stages [stages][2 k-halves][128 x 128 B],
// then B [2 k-halves][c_pad x 128 B], then the barriers.  B is the resident
// operand for one unit; A (key tiles) streams.
struct TcBars {
  uint64_t a_full[4], a_empty[4];
  uint64_t b_full, b_empty;
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
  uint32_t pad_[3];
  // epilogue exchange, [..][row] so a warp's accesses are conflict-free
  float m_part[TC_EGROUPS][TC_M];         // per-group max of the current chunk
  float m_ch[2][TC_M];                    // chunk maxima of the current tile
  uint32_t n_ch[2][TC_M];                 // in-band columns per chunk
  uint16_t id_ch[2][TC_NCAND][TC_M];      // their ids (first TC_NCAND)
  uint32_t fix_n;                         // this CTA's fix-up entries
};
constexpr uint32_t TC_ABYTES = TC_M * 128 * 2;  // one key-tile stage (both k-halves)
constexpr uint32_t TC_BOXR = 32;                // rows per B TMA box (B sized to c_pad)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
// Watchdog for the pipelines' barrier waits: a wait still unsatisfied after
// ~4 s of device time reports the barrier and traps, so a pipeline bug ends
// the launch with an error instead of hanging the device.
__device__ __noinline__ void mb_wait_timeout(const uint64_t* b, uint32_t parity) {
  printf("[ckv] mbarrier wait timed out: block %d thread %d barrier smem+%u parity %u\n",
         int(blockIdx.x), int(threadIdx.x), su32(b), parity);
  __trap();
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct MbWatch {
  uint32_t n = 0;
  uint64_t t0 = 0;
  __device__ __forceinline__ void tick(const uint64_t* b, uint32_t parity) {
    if ((++n & 4095u) == 0u) {
      const uint64_t t = global_ns();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 4000000000ull) mb_wait_timeout(b, parity);
    }
  }
};
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  MbWatch wd;
  for (;;) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(su32(b)), "r"(parity) : "memory");
    if (done) break;
    wd.tick(b, parity);
  }
}
// bit 31-j of the result set <=> x[j] < lo (the sign of the rounded x[j] - lo;
// x[j] >= lo gives a difference >= +0).  FADD2 + four interleaved SHF chains.
__device__ __forceinline__ uint32_t below_mask32(const float* x, float lo) {
  uint32_t b[4] = {0u, 0u, 0u, 0u};
  unsigned long long l2;
  asm("mov.b64 %0, {%1, %1};" : "=l"(l2) : "f"(lo));
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      unsigned long long a2, d2;
      asm("mov.b64 %0, {%1, %2};" : "=l"(a2) : "f"(x[8 * c + j]), "f"(x[8 * c + j + 1]));
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d2) : "l"(a2), "l"(l2));
      uint32_t r0, r1;
      asm("mov.b64 {%0, %1}, %2;" : "=r"(r0), "=r"(r1) : "l"(d2));
      b[c] = __funnelshift_l(r0, b[c], 1);
      b[c] = __funnelshift_l(r1, b[c], 1);
    }
  }
  // b[c] holds x[8c .. 8c+7] in bits 7..0: word = b0.b1.b2.b3 (bytes, high first)
  return __byte_perm(__byte_perm(b[3], b[2], 0x0040), __byte_perm(b[1], b[0], 0x0040), 0x5410);
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
// K-major, SWIZZLE_128B smem matrix descriptor (tcgen05 "version 1"):
// start >> 4 | LBO (unused for swizzled K-major) = 1 | SBO = 1024 B (8 rows)
__device__ __forceinline__ uint64_t kmajor_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3fff);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;  // version
  d |= uint64_t(2) << 61;  // SWIZZLE_128B
  return d;
}
// instruction descriptor: kind::f16, A/B f16 (format 0), D f32, K-major A and B
__host__ __device__ constexpr uint32_t idesc_f16_f32(uint32_t M, uint32_t N) {
  return (1u << 4) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; "
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                   "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// 32 lanes x 32 bit, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 bit, 32 consecutive columns per thread, no wait (pair with
// tmem_wait so several loads are in flight)
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 32 lanes x 32 bit, 32 consecutive columns per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct TcArgs {
  uint32_t stages;           // key-tile stages that fit next to B
  const int32_t* unit_list;  // active units
  const int32_t* n_list;     // device count of active units
  uint32_t n, C, c_pad, tiles_per_unit;
  // C > 512: the columns split into n_ranges ranges of rc (a multiple of 32,
  // <= 512) columns, each its own work item with a resident B; the epilogue
  // then writes a per-(key, range) summary and k_assign_merge decides
  uint32_t n_ranges, rc;
  float4* summ;                // [unit][n][n_slots]: M_r, n_in | FULL, 4 ids (u16)
  uint32_t n_slots;            // summary slots per key (n_ranges, or the work list's)
  // explicit work list (the moved-cluster pass, ckv_assign_mcr.cu): item =
  // {unit, tile, first column, columns | slot << 16}; summaries only
  const uint4* wlist;
  const int32_t* n_wlist;
  uint32_t key_rows_per_unit;  // key_stride / 128
  uint32_t label_stride;
  const float* knorm;          // [unit][n] key norms (band scale)
  const float* eps_u;          // [unit] max_c |dir_c - h(dir_c)|
  const float* kerr_u;         // [unit] max_k |k - h(k)| (k_scan_keys)
  int32_t* labels;
  uint32_t* fix_count;         // [gridDim.x] per-CTA fix-up counts (region = w0 * 128)
  uint4* fix_list;             // {unit, row, n_cand | FULL, 0}
  uint32_t fix_cap;
  uint32_t* fix_ids;           // [fix_cap][8] candidate ids
  // k16 rows in cluster-major order (k_permute_keys): row r of the A operand
  // is key position perm[unit][r]; nullptr = position order
  const uint32_t* perm;
  uint32_t mode;               // experiment knob (CKV_TC_MODE): 1 = no epilogue math,
                               // 2 = no TMEM reads either (producer + MMA only)
};

// the score band of a key (see the header): twice one score's error bound
__device__ __forceinline__ float tc_band(float kn, float eps, float kerr) {
  return kn * (2.0f * eps + (1.0f / 8192.0f)) * 1.01f + 2.02f * kerr + 1e-30f;
}

struct TcWork {
  uint32_t ui, range, tile;
};
__device__ __forceinline__ TcWork tc_work(uint32_t w, const TcArgs& a) {
  const uint32_t per_u = a.n_ranges * a.tiles_per_unit;
  TcWork k;
  k.ui = w / per_u;
  const uint32_t r = w - k.ui * per_u;
  k.range = r / a.tiles_per_unit;
  k.tile = r - k.range * a.tiles_per_unit;
  return k;
}
__device__ __forceinline__ uint32_t tc_cols(uint32_t range, const TcArgs& a) {
  return min(a.rc, a.c_pad - range * a.rc);
}
// one work item: a 128-key tile of `unit` against columns [cbeg, cbeg + ccnt)
struct TcItem {
  uint32_t unit, tile, cbeg, ccnt, slot;
};
__device__ __forceinline__ TcItem tc_item_of(const TcWork& k, const TcArgs& a) {
  return TcItem{uint32_t(a.unit_list[k.ui]), k.tile, k.range * a.rc, tc_cols(k.range, a),
                k.range};
}
__device__ __forceinline__ TcItem tc_item(uint32_t w, const TcArgs& a) {
  if (a.wlist) {
    const uint4 x = a.wlist[w];
    return TcItem{x.x, x.y, x.z, x.w & 0xffffu, x.w >> 16};
  }
  return tc_item_of(tc_work(w, a), a);
}

__global__ void __launch_bounds__(TC_THREADS, 1)
k_assign_tc(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap dmap,
            TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sbase = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const uint32_t S = a.stages;
  uint8_t* sm_a = sbase;                         // [S][2][TC_M*128]
  uint8_t* sm_b = sbase + S * TC_ABYTES;         // [2][rc*128]
  __shared__ TcBars sm;  // static: the compiler keeps these accesses LDS/STS
  auto A = [&](uint32_t st, uint32_t kh) { return sm_a + st * TC_ABYTES + kh * (TC_M * 128); };
  auto Bp = [&](uint32_t kh, uint32_t row) { return sm_b + kh * (a.rc * 128) + row * 128; };
  const int t = threadIdx.x, wid = t >> 5, lane = t & 31;
  const uint32_t n_units = uint32_t(*a.n_list);
  const uint32_t total = a.wlist ? uint32_t(*a.n_wlist) : n_units * a.n_ranges * a.tiles_per_unit;
  const bool summary = a.summ && (a.n_ranges > 1 || a.wlist);
  const uint32_t per = (total + gridDim.x - 1) / gridDim.x;
  const uint32_t w0 = min(total, blockIdx.x * per), w1 = min(total, w0 + per);

  if (t == 0) {
    for (uint32_t s = 0; s < S; ++s) { mb_init(&sm.a_full[s], 1); mb_init(&sm.a_empty[s], 1); }
    mb_init(&sm.b_full, 1);
    mb_init(&sm.b_empty, 1);
    for (int s = 0; s < 2; ++s) { mb_init(&sm.acc_full[s], 1); mb_init(&sm.acc_empty[s], 4 * TC_EGROUPS); }
    sm.fix_n = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (wid == 1) {  // TMEM: 512 columns (two 256-column accumulator buffers)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     su32(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (wid == 0) {
    // ============================ TMA producer =================================
    if (lane == 0 && w0 < w1) {
      uint32_t st = 0, ph = 0, bswitch = 0;
      unsigned long long cur_key = ~0ull;
      for (uint32_t w = w0; w < w1; ++w) {
        const TcItem it = tc_item(w, a);
        const uint32_t tile = it.tile, unit = it.unit;
        const unsigned long long key = (unsigned long long)unit << 32 | it.cbeg;
        if (key != cur_key) {
          // the previous (unit, columns)'s MMAs must be done reading B
          if (cur_key != ~0ull) mb_wait(&sm.b_empty, (bswitch - 1) & 1);
          const uint32_t cols = it.ccnt;  // a multiple of TC_BOXR
          mb_expect(&sm.b_full, cols * 128 * 2);
          for (uint32_t r0 = 0; r0 < cols; r0 += TC_BOXR) {
            for (int kh = 0; kh < 2; ++kh)
              tma_2d(Bp(kh, r0), &dmap, kh * TC_BK, int(unit * a.c_pad + it.cbeg + r0),
                     &sm.b_full);
          }
          cur_key = key;
          ++bswitch;
        }
        mb_wait(&sm.a_empty[st], ph ^ 1);
        mb_expect(&sm.a_full[st], TC_ABYTES);
        const int row = int(unit * a.key_rows_per_unit + tile * TC_M);
        tma_2d(A(st, 0), &kmap, 0, row, &sm.a_full[st]);
        tma_2d(A(st, 1), &kmap, TC_BK, row, &sm.a_full[st]);
        if (++st == S) { st = 0; ph ^= 1; }
      }
    }
  } else if (wid == 1) {
    // ============================ MMA issuer ===================================
    if (lane == 0 && w0 < w1) {
      uint32_t st = 0, ph = 0, g = 0, bswitch = 0;
      unsigned long long cur_key = ~0ull;
      for (uint32_t w = w0; w < w1; ++w) {
        const TcItem it = tc_item(w, a);
        const unsigned long long key = (unsigned long long)it.unit << 32 | it.cbeg;
        bool last_of_unit = w + 1 == w1;
        if (!last_of_unit) {
          const TcItem nx = tc_item(w + 1, a);
          last_of_unit = ((unsigned long long)nx.unit << 32 | nx.cbeg) != key;
        }
        if (key != cur_key) {
          mb_wait(&sm.b_full, bswitch & 1);
          cur_key = key;
          ++bswitch;
        }
        mb_wait(&sm.a_full[st], ph);
        tc_fence_after();
        const uint32_t cols = it.ccnt;
        const uint32_t nchunks = (cols + TC_CH - 1) / TC_CH;
        for (uint32_t ch = 0; ch < nchunks; ++ch, ++g) {
          const uint32_t buf = g & 1, bph = (g >> 1) & 1;
          const uint32_t c0 = ch * TC_CH;
          const uint32_t nc = min(uint32_t(TC_CH), cols - c0);
          mb_wait(&sm.acc_empty[buf], bph ^ 1);
          tc_fence_after();
          const uint32_t idesc = idesc_f16_f32(TC_M, nc);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int kh = kk >> 2, ko = (kk & 3) * 32;  // 16 halves = 32 B per K step
            const uint64_t ad = kmajor_sw128_desc(su32(A(st, kh)) + ko);
            const uint64_t bd = kmajor_sw128_desc(su32(Bp(kh, c0)) + ko);
            umma_f16(tmem + buf * TC_CH, ad, bd, idesc, kk > 0 ? 1u : 0u);
          }
          umma_commit(&sm.acc_full[buf]);
        }
        umma_commit(&sm.a_empty[st]);  // key tile consumed once these MMAs finish
        if (last_of_unit) umma_commit(&sm.b_empty);
        if (++st == S) { st = 0; ph ^= 1; }
      }
    }
  } else {
    // ============================ epilogue =====================================
    // 16 warps: 4 per TMEM lane quarter (one key row per thread), splitting
    // each chunk's 32-column blocks round-robin, <= 2 blocks each, held in
    // registers after ONE tcgen05.ld pass, so the buffer is released at once.
    // Per chunk: (1) block maxima -> m_part; named barrier of the quarter;
    // (2) chunk max M_ch = max of the 4 parts; in-band mask S >= M_ch - band
    // per block; the (rare) in-band ids go to the row's chunk list; barrier.
    // After the tile's last chunk the quarter's last warp decides each row:
    // M = max_ch M_ch; the chunks with M_ch >= M - band contribute their
    // in-band ids (a superset of {c : S_c >= M - band}; it only differs when
    // two chunks are both in band, i.e. the row has >= 2 candidates anyway).
    const uint32_t quarter = wid & 3;               // TMEM lanes [32q, 32q+32)
    const uint32_t grp = uint32_t(wid - 2) >> 2;    // 0..3: column share
    const uint32_t lane_row = quarter * 32 + lane;
    const uint32_t bar_id = 1 + quarter;            // named barrier per quarter
    // the group that records chunk maxima and decides each row after the
    // tile: the last one, which holds the fewest blocks of a partial last
    // chunk (blocks are dealt round-robin from group 0)
    constexpr uint32_t kDecider = TC_EGROUPS - 1;
    auto qbar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(4 * 32) : "memory"); };
    uint32_t g = 0;
    if (grp == kDecider)
      for (int ch = 0; ch < 2; ++ch) sm.n_ch[ch][lane_row] = 0;
    // (unit, range, tile) advance incrementally (no integer divisions per
    // item).  The NEXT item is resolved one item ahead: its unit id and eps
    // are re-read only when the unit changes (every tiles_per_unit x n_ranges
    // items; otherwise the unit_list -> eps_u / knorm loads form a dependent
    // global chain on every item), and its key norm load is issued one item
    // before it is used so the latency hides behind this item's chunks.
    TcWork nx = tc_work(w0, a);
    auto advance = [&](TcWork& k) {
      if (++k.tile == a.tiles_per_unit) {
        k.tile = 0;
        if (++k.range == a.n_ranges) { k.range = 0; ++k.ui; }
      }
    };
    uint32_t nx_ui = ~0u;
    TcItem itn = TcItem{0, 0, 0, 0, 0};
    float kn_next = 0.f, eps_next = 0.f, kerr_next = 0.f;
    auto resolve_next = [&](uint32_t w) {
      if (a.wlist) {
        itn = tc_item(w, a);
        eps_next = a.eps_u[itn.unit];
        kerr_next = a.kerr_u[itn.unit];
      } else {
        if (nx.ui != nx_ui) {
          nx_ui = nx.ui;
          itn.unit = uint32_t(a.unit_list[nx.ui]);
          eps_next = a.eps_u[itn.unit];
          kerr_next = a.kerr_u[itn.unit];
        }
        itn.tile = nx.tile;
        itn.cbeg = nx.range * a.rc;
        itn.ccnt = tc_cols(nx.range, a);
        itn.slot = nx.range;
      }
      const uint32_t r2 = itn.tile * TC_M + lane_row;
      kn_next = r2 < a.n ? a.knorm[size_t(itn.unit) * a.n + r2] : 0.f;
    };
    if (w0 < w1) resolve_next(w0);
    for (uint32_t w = w0; w < w1; ++w) {
      const TcItem it = itn;
      const float eps = eps_next, kn = kn_next, kerr = kerr_next;
      const uint32_t unit = it.unit, tile = it.tile;
      const uint32_t row = tile * TC_M + lane_row;
      if (w + 1 < w1) {
        if (!a.wlist) advance(nx);
        resolve_next(w + 1);
      }
      const float band = tc_band(kn, eps, kerr);
      const uint32_t cols = it.ccnt, cbase = it.cbeg;
      const uint32_t nchunks = (cols + TC_CH - 1) / TC_CH;
#pragma unroll 1
      for (uint32_t ch = 0; ch < nchunks; ++ch) {
        const uint32_t buf = g & 1, bph = (g >> 1) & 1;
        ++g;
        const uint32_t c0 = cbase + ch * TC_CH;  // global column of the chunk
        const uint32_t nb = min(uint32_t(TC_CH), cols - ch * TC_CH) / 32;  // blocks in chunk
        const uint32_t b0 = grp, b1 = grp + TC_EGROUPS;               // my blocks
        const bool h0 = b0 < nb, h1 = b1 < nb;                         // warp-uniform
        float v[64];
        mb_wait(&sm.acc_full[buf], bph);
        tc_fence_after();
        if (a.mode == 2) {  // experiment: producer + MMA rate only
          __syncwarp();
          if (lane == 0) mb_arrive(&sm.acc_empty[buf]);
          if (grp == kDecider) sm.m_ch[ch][lane_row] = 0.f;
          continue;
        }
        const uint32_t taddr = tmem + ((quarter * 32) << 16) + buf * TC_CH;
        if (h0) tmem_ld32_nw(taddr + b0 * 32, v);
        if (h1) tmem_ld32_nw(taddr + b1 * 32, v + 32);
        tmem_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mb_arrive(&sm.acc_empty[buf]);  // scores now live in registers
        const uint32_t cb0 = c0 + b0 * 32, cb1 = c0 + b1 * 32;
        if (a.mode == 1) {
          if (grp == kDecider) sm.m_ch[ch][lane_row] = 0.f;
          qbar();
          qbar();
          continue;
        }
        // padding columns (only in the unit's last block; warp-uniform branch)
        if (h0 && cb0 + 32 > a.C) {
#pragma unroll
          for (int j = 0; j < 32; ++j) if (cb0 + j >= a.C) v[j] = -INFINITY;
        }
        if (h1 && cb1 + 32 > a.C) {
#pragma unroll
          for (int j = 0; j < 32; ++j) if (cb1 + j >= a.C) v[32 + j] = -INFINITY;
        }
        // (1) block maximum: FMNMX3 trees (ALU pipe, 0.5 op per score)
        float mx = -INFINITY;
        if (h1) {
          float t[16];
#pragma unroll
          for (int j = 0; j < 16; ++j)
            t[j] = fmaxf(fmaxf(v[j], v[j + 16]), fmaxf(v[j + 32], v[j + 48]));
#pragma unroll
          for (int w2 = 8; w2 > 0; w2 >>= 1)
#pragma unroll
            for (int j = 0; j < w2; ++j) t[j] = fmaxf(t[j], t[j + w2]);
          mx = t[0];
        } else if (h0) {
          float t[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) t[j] = fmaxf(v[j], v[j + 16]);
#pragma unroll
          for (int w2 = 8; w2 > 0; w2 >>= 1)
#pragma unroll
            for (int j = 0; j < w2; ++j) t[j] = fmaxf(t[j], t[j + w2]);
          mx = t[0];
        }
        sm.m_part[grp][lane_row] = mx;
        qbar();
        float mc = sm.m_part[0][lane_row];
#pragma unroll
        for (int q = 1; q < TC_EGROUPS; ++q) mc = fmaxf(mc, sm.m_part[q][lane_row]);
        if (grp == kDecider) sm.m_ch[ch][lane_row] = mc;
        // band relative to the running max of the tile's chunks so far: a
        // later chunk far below an earlier one contributes no candidates
        // (still a superset of {c : S_c >= M - band}, M the final max)
        const float lo = (ch > 0 ? fmaxf(mc, sm.m_ch[0][lane_row]) : mc) - band;
        // (2) in-band mask: sign of S - lo (FADD2, two scores per FMA-pipe op)
        // funnel-shifted into a word (SHF, ALU pipe): bit 31-j set <=> S_j < lo.
        // Four independent 8-bit chains per block (joined by PRMT) so the
        // shifts do not form one 32-long dependency chain; both blocks' chains
        // sit in one basic block so they interleave.
        uint32_t in0 = 0u, in1 = 0u;
        if (h1) {
          in0 = ~below_mask32(v, lo);
          in1 = ~below_mask32(v + 32, lo);
        } else if (h0) {
          in0 = ~below_mask32(v, lo);
        }
        // (3) the rare in-band columns -> the row's chunk list
        while (in0 | in1) {
          const bool first = in0 != 0u;
          const uint32_t word = first ? in0 : in1;
          const uint32_t jj = __clz(word);
          const uint32_t c = (first ? cb0 : cb1) + jj;
          if (first) in0 &= ~(0x80000000u >> jj); else in1 &= ~(0x80000000u >> jj);
          const uint32_t slot = atomicAdd(&sm.n_ch[ch][lane_row], 1u);
          if (slot < uint32_t(TC_NCAND)) sm.id_ch[ch][slot][lane_row] = uint16_t(c);
        }
        qbar();
      }
      if (grp == kDecider) {
        if (row < a.n && a.mode == 0) {
          float M = sm.m_ch[0][lane_row];
          if (nchunks > 1) M = fmaxf(M, sm.m_ch[1][lane_row]);
          bool full = !(M > -INFINITY);
          uint32_t nin = 0, single = TC_FULL;
          for (uint32_t ch = 0; ch < nchunks; ++ch) {
            if (sm.m_ch[ch][lane_row] >= M - band) {
              const uint32_t nn = sm.n_ch[ch][lane_row];
              if (nn > uint32_t(TC_NCAND)) full = true;
              if (nn > 0) single = sm.id_ch[ch][0][lane_row];
              nin += nn;
            }
          }
          if (nin > uint32_t(TC_NCAND)) full = true;
          int32_t* lab = a.labels + size_t(unit) * a.label_stride + row;
          if (summary) {
            // this range's summary: its max and its (<= 4) in-band ids;
            // k_assign_merge combines the ranges of the key
            uint32_t ids[4] = {0u, 0u, 0u, 0u}, k2 = 0;
            if (nin > 4u) full = true;
            if (!full)
              for (uint32_t ch = 0; ch < nchunks; ++ch)
                if (sm.m_ch[ch][lane_row] >= M - band)
                  for (uint32_t k = 0; k < sm.n_ch[ch][lane_row]; ++k)
                    ids[k2++] = sm.id_ch[ch][k][lane_row];
            a.summ[(size_t(unit) * a.n + row) * a.n_slots + it.slot] =
                make_float4(M, __uint_as_float(full ? TC_FULL : nin),
                            __uint_as_float(ids[0] | (ids[1] << 16)),
                            __uint_as_float(ids[2] | (ids[3] << 16)));
          } else if (!full && nin == 1) {
            *lab = int32_t(single);
          } else {
            *lab = -1;
            // this CTA's region of the list: a shared-memory counter, no
            // device-wide atomic (one hot address across all SMs serialises)
            const uint32_t slot = w0 * TC_M + atomicAdd(&sm.fix_n, 1u);
            if (slot < a.fix_cap) {
              a.fix_list[slot] = make_uint4(unit, row, full ? TC_FULL : nin, 0u);
              uint32_t* fi = a.fix_ids + size_t(slot) * TC_NCAND;
              uint32_t k2 = 0;
              if (!full)
                for (uint32_t ch = 0; ch < nchunks; ++ch)
                  if (sm.m_ch[ch][lane_row] >= M - band)
                    for (uint32_t k = 0; k < sm.n_ch[ch][lane_row]; ++k)
                      fi[k2++] = sm.id_ch[ch][k][lane_row];
            }
          }
        }
        __syncwarp();
        for (int ch = 0; ch < 2; ++ch) sm.n_ch[ch][lane_row] = 0;
      }
    }
  }
  __syncthreads();
  if (t == 0) a.fix_count[blockIdx.x] = sm.fix_n;
  if (wid == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ===========================================================================
// k_assign_tc2: the same assignment filter with a barrier-free epilogue.
//
// k_assign_tc's 16 epilogue warps split each chunk's columns, so every row's
// maximum needs two named barriers per chunk and one warp decides all rows
// after the tile: the epilogue, not the tensor pipe, set the pass time.
// Here the epilogue warps split TILES, not columns:
//   * T2_CG epilogue warps per TMEM lane quarter; warp g takes the items
//     s = g, g + CG, ... of the CTA, and each of its threads owns one key row
//     across ALL columns of the item, so the row's decision needs no exchange
//     with any other warp (no barrier, no shared state);
//   * per row the thread keeps an exact running state: the two best entries
//     {score, first column, in-band mask of a 32-column block} and the
//     largest score displaced from them.  A block's entry lists its columns
//     >= (running max - band) with the block maximum as their score;
//   * accumulator chunks are 256 columns (two TMEM buffers): the SS-mode MMA
//     re-reads the A tile from shared memory once per chunk, and at K = 128
//     the shared-memory operand traffic bounds the producer + MMA rate
//     (measured: 128-column chunks cost 1.5x).  A warp reads a chunk in
//     groups of 4 blocks (128 registers) and releases it after the last
//     group's loads; the other warp of the quarter works on the next item
//     meanwhile.
// Exactness: a column c with S_c >= M - band is >= (running max - band) when
// its block is scanned (the running max never exceeds M), so it enters an
// entry; it can only leave by being displaced, which records a dropped score
// >= S_c.  Listed scores are upper bounds of the true S, so the final filter
// (entries with score >= M - band) is a superset of {c : S_c >= M - band} --
// which contains the exact argmax (see the header) -- and a single survivor
// is the label.  Padding columns (>= C) score exactly 0 (zero operand rows);
// a surviving one makes the row FULL (exact fix-up over all C).
// ===========================================================================
#ifndef CKV_T2_ENTRIES
#define CKV_T2_ENTRIES 4  // in-band entries per row: 2 scored + 2 bounded by e1, or 2
#endif
constexpr int T2_CW = 256;                       // columns per TMEM chunk buffer
constexpr int T2_NBUF = 512 / T2_CW;             // chunk buffers (512 TMEM columns)
constexpr int T2_CG = T2_NBUF;                   // epilogue warps per lane quarter: one per buffer
#ifndef CKV_T2_GB
#define CKV_T2_GB 2
#endif
constexpr int T2_GB = CKV_T2_GB;                 // blocks a warp holds in registers at once
constexpr int T2_THREADS = (2 + 4 * T2_CG) * 32;
struct T2Bars {
  uint64_t a_full[4], a_empty[4];
  uint64_t b_full, b_empty;
  // TMEM buffer g belongs to epilogue group g (items of parity g)
  uint64_t acc_full[T2_NBUF][1], acc_empty[T2_NBUF];
  uint32_t tmem_base;
  uint32_t fix_n;
};
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}


// Waits that back off with __nanosleep between probes: a spinning single-
// thread producer / MMA warp otherwise issues a probe every few cycles on
// the same SM sub-partition as two column warps (measured: 22% of the
// kernel's instructions).  The MMA thread sleeps briefly (its wake-up delay
// hides under the chunk the tensor pipe is still computing), the producer
// longer (it runs stages ahead).
template <uint32_t NS>
__device__ __forceinline__ void mb_wait_sleep(uint64_t* b, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(done) : "r"(su32(b)), "r"(parity) : "memory");
  MbWatch wd;
  while (!done) {
    __nanosleep(NS);
    wd.tick(b, parity);
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(su32(b)), "r"(parity) : "memory");
  }
}
#ifndef CKV_T2_NS_MMA
#define CKV_T2_NS_MMA 64
#endif
#ifndef CKV_T2_NS_PROD
#define CKV_T2_NS_PROD 256
#endif
#ifndef CKV_T2_NS_EPI
#define CKV_T2_NS_EPI 0
#endif
__device__ __forceinline__ void mb_wait_epi(uint64_t* b, uint32_t parity) {
  if (CKV_T2_NS_EPI > 0) mb_wait_sleep<CKV_T2_NS_EPI>(b, parity); else mb_wait(b, parity);
}
__device__ __forceinline__ void mb_wait_mma(uint64_t* b, uint32_t parity) {
  mb_wait_sleep<CKV_T2_NS_MMA>(b, parity);
}
__device__ __forceinline__ void mb_wait_prod(uint64_t* b, uint32_t parity) {
  mb_wait_sleep<CKV_T2_NS_PROD>(b, parity);
}
// CKV_T2_PROF builds: cycles each role spends in its waits, summed over CTAs
// ([0] producer a_empty, [1] MMA a_full, [2] MMA acc_empty, [3] epilogue
// acc_full, [5] MMA b_full, [6] kernel cycles, [7] epilogue warp lifetime),
// printed after every launch by t2_prof_dump()
#ifdef CKV_T2_PROF
__device__ unsigned long long g_t2prof[8];
#define T2P_BEGIN(v) const long long v = clock64();
#define T2P_END(v, slot) acc_[slot] += clock64() - v;
#else
#define T2P_BEGIN(v)
#define T2P_END(v, slot)
#endif

// 10 warps: 3 share an SM sub-partition's 16K-register file, so <= 168 registers
__global__ void __launch_bounds__(T2_THREADS, 1)
k_assign_tc2(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap dmap,
             TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sbase = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const uint32_t S = a.stages;
  uint8_t* sm_a = sbase;                         // [S][2][TC_M*128]
  uint8_t* sm_b = sbase + S * TC_ABYTES;         // [2][rc*128]
  __shared__ T2Bars sm;
  auto A = [&](uint32_t st, uint32_t kh) { return sm_a + st * TC_ABYTES + kh * (TC_M * 128); };
  auto Bp = [&](uint32_t kh, uint32_t row) { return sm_b + kh * (a.rc * 128) + row * 128; };
  const int t = threadIdx.x, wid = t >> 5, lane = t & 31;
#ifdef CKV_T2_PROF
  unsigned long long acc_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long tk0_ = clock64();
#endif
  const uint32_t n_units = uint32_t(*a.n_list);
  const uint32_t total = n_units * a.n_ranges * a.tiles_per_unit;
  const bool summary = a.summ && a.n_ranges > 1;
  const uint32_t per = (total + gridDim.x - 1) / gridDim.x;
  const uint32_t w0 = min(total, blockIdx.x * per), w1 = min(total, w0 + per);
  auto next_work = [&](TcWork& k) {
    if (++k.tile == a.tiles_per_unit) {
      k.tile = 0;
      if (++k.range == a.n_ranges) { k.range = 0; ++k.ui; }
    }
  };

  if (t == 0) {
    for (uint32_t s = 0; s < S; ++s) { mb_init(&sm.a_full[s], 1); mb_init(&sm.a_empty[s], 1); }
    mb_init(&sm.b_full, 1);
    mb_init(&sm.b_empty, 1);
    // one consuming warp per lane quarter per chunk
    for (int s = 0; s < T2_NBUF; ++s) { mb_init(&sm.acc_full[s][0], 1); mb_init(&sm.acc_empty[s], 4); }
    sm.fix_n = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (wid == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     su32(&sm.tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (wid == 0) {
    // ============================ TMA producer =================================
    if (lane == 0 && w0 < w1) {
      uint32_t st = 0, ph = 0, bswitch = 0;
      unsigned long long cur_key = ~0ull;
      TcWork k = tc_work(w0, a);
      uint32_t unit = uint32_t(a.unit_list[k.ui]), cur_ui = k.ui;
      for (uint32_t w = w0; w < w1; ++w) {
        if (k.ui != cur_ui) { cur_ui = k.ui; unit = uint32_t(a.unit_list[k.ui]); }
        const uint32_t cbeg = k.range * a.rc;
        const unsigned long long key = (unsigned long long)unit << 32 | cbeg;
        // the key tile first: at a B switch it streams in while the last
        // MMAs on the old B drain
        T2P_BEGIN(t0_) mb_wait_prod(&sm.a_empty[st], ph ^ 1); T2P_END(t0_, 0)
        mb_expect(&sm.a_full[st], TC_ABYTES);
        const int row = int(unit * a.key_rows_per_unit + k.tile * TC_M);
        tma_2d(A(st, 0), &kmap, 0, row, &sm.a_full[st]);
        tma_2d(A(st, 1), &kmap, TC_BK, row, &sm.a_full[st]);
        if (key != cur_key) {
          if (cur_key != ~0ull) mb_wait_prod(&sm.b_empty, (bswitch - 1) & 1);
          const uint32_t cols = tc_cols(k.range, a);
          mb_expect(&sm.b_full, cols * 128 * 2);
          for (uint32_t r0 = 0; r0 < cols; r0 += TC_BOXR)
            for (int kh = 0; kh < 2; ++kh)
              tma_2d(Bp(kh, r0), &dmap, kh * TC_BK, int(unit * a.c_pad + cbeg + r0), &sm.b_full);
          cur_key = key;
          ++bswitch;
        }
        if (++st == S) { st = 0; ph ^= 1; }
        next_work(k);
      }
    }
  } else if (wid == 1) {
    // ============================ MMA issuer ===================================
    // Items alternate between the two epilogue groups (item parity) and group
    // g owns TMEM buffer g.  Consecutive items on the same B are issued as a
    // pair with their chunks interleaved (A_w, A_w+1, B_w, B_w+1, ...), so the
    // tensor pipe works for one group while the other drains its buffer.
    if (lane == 0 && w0 < w1) {
      uint32_t st = 0, ph = 0, bswitch = 0, ue0 = 0, ue1 = 0;
      unsigned long long cur_key = ~0ull;
      TcWork k = tc_work(w0, a);
      uint32_t unit = uint32_t(a.unit_list[k.ui]), cur_ui = k.ui;
      auto key_of = [&](const TcWork& kw, uint32_t u) {
        return (unsigned long long)u << 32 | (kw.range * a.rc);
      };
      for (uint32_t w = w0; w < w1;) {
        if (k.ui != cur_ui) { cur_ui = k.ui; unit = uint32_t(a.unit_list[k.ui]); }
        const unsigned long long key = key_of(k, unit);
        TcWork k2 = k;
        next_work(k2);
        // the pair shares B: same unit and column range (a tile change only)
        const bool pair = w + 1 < w1 && k2.tile != 0;
        TcWork k3 = k2;
        if (pair) next_work(k3);
        const uint32_t nit = pair ? 2u : 1u;
        // last items on this B: the item after them changes the range or unit
        const bool last_b = w + nit >= w1 || (pair ? k3.tile == 0 : k2.tile == 0);
        if (key != cur_key) {
          T2P_BEGIN(t0_) mb_wait_mma(&sm.b_full, bswitch & 1); T2P_END(t0_, 5)
          cur_key = key;
          ++bswitch;
        }
        const uint32_t cols = tc_cols(k.range, a);
        uint32_t stq[2];
        for (uint32_t x = 0; x < nit; ++x) {
          stq[x] = st;
          T2P_BEGIN(t1_) mb_wait_mma(&sm.a_full[st], ph); T2P_END(t1_, 1)
          if (++st == S) { st = 0; ph ^= 1; }
        }
        tc_fence_after();
        for (uint32_t c0 = 0; c0 < cols; c0 += T2_CW) {
          const uint32_t nc = min(uint32_t(T2_CW), cols - c0);
          const uint32_t idesc = idesc_f16_f32(TC_M, nc);
          for (uint32_t x = 0; x < nit; ++x) {
            const uint32_t buf = (w + x - w0) & 1;
            const uint32_t bph = ((buf ? ue1 : ue0) & 1) ^ 1;
            if (buf) ++ue1; else ++ue0;
            T2P_BEGIN(t2_) mb_wait_mma(&sm.acc_empty[buf], bph); T2P_END(t2_, 2)
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const int kh = kk >> 2, ko = (kk & 3) * 32;
              const uint64_t ad = kmajor_sw128_desc(su32(A(stq[x], kh)) + ko);
              const uint64_t bd = kmajor_sw128_desc(su32(Bp(kh, c0)) + ko);
              umma_f16(tmem + buf * T2_CW, ad, bd, idesc, kk > 0 ? 1u : 0u);
            }
            umma_commit(&sm.acc_full[buf][0]);
          }
        }
        for (uint32_t x = 0; x < nit; ++x) umma_commit(&sm.a_empty[stq[x]]);
        if (last_b) umma_commit(&sm.b_empty);
        w += nit;
        k = pair ? k3 : k2;
      }
    }
  } else {
    // ============================ epilogue warps ===============================
    const uint32_t quarter = wid & 3, grp = uint32_t(wid - 2) >> 2;
    const uint32_t lane_row = quarter * 32 + lane;
    const uint32_t tq = tmem + ((quarter * 32) << 16);
    TcWork k = tc_work(w0, a);
    uint32_t uses = 0;  // chunks of this group so far (acc_full phases of buffer grp)
    uint32_t cur_ui = ~0u, unit = 0;
    float eps = 0.f, kerr = 0.f;
    if (grp == 1) next_work(k);  // this warp's first item
    for (uint32_t w = w0 + grp; w < w1; w += T2_CG) {
      const uint32_t cols = tc_cols(k.range, a);
      const uint32_t nch = (cols + T2_CW - 1) / T2_CW;
      if (k.ui != cur_ui) {
        cur_ui = k.ui;
        unit = uint32_t(a.unit_list[k.ui]);
        eps = a.eps_u[unit];
        kerr = a.kerr_u[unit];
      }
      const uint32_t prow = k.tile * TC_M + lane_row, cbeg = k.range * a.rc, range = k.range;
      // the key position of this A row (cluster-major operand after k_permute_keys)
      const uint32_t row = a.perm ? __ldg(a.perm + size_t(unit) * a.key_rows_per_unit + prow) : prow;
      // issued now, first used after the accumulator wait (which hides it);
      // rows past n: a negative band admits no candidate (lo > block max)
      const float kn = row < a.n ? __ldg(a.knorm + size_t(unit) * a.n + row) : -1.f;
      float band = 0.f;
      // two best entries {score, first column, in-band mask} and the largest
      // score displaced from them
      float e0s = -INFINITY, e1s = -INFINITY, dmax = -INFINITY;
      uint32_t e0c = 0u, e0m = 0u, e1c = 0u, e1m = 0u, e2c = 0u, e2m = 0u, e3c = 0u, e3m = 0u;
#pragma unroll 1
      for (uint32_t ch = 0; ch < nch; ++ch) {
        const uint32_t cc = ch * T2_CW;
        const uint32_t nbk = min(uint32_t(T2_CW), cols - cc) / 32;
        const uint32_t buf = grp, bph = uses++ & 1;
        T2P_BEGIN(t0_) mb_wait_epi(&sm.acc_full[buf][0], bph); T2P_END(t0_, 3)
        tc_fence_after();
        if (ch == 0) band = kn < 0.f ? -1.f : tc_band(kn, eps, kerr);
        if (a.mode == 2) {
          __syncwarp();
          if (lane == 0) mb_arrive(&sm.acc_empty[buf]);
          continue;
        }
        const uint32_t taddr = tq + buf * T2_CW;
#pragma unroll 1
        for (uint32_t b0 = 0; b0 < nbk; b0 += T2_GB) {
          // T2_GB blocks in registers at once; a slot past the chunk's last
          // block re-reads it and is masked out, so the code is straight-line
          // (no per-block branches: the blocks' chains interleave)
          float v[T2_GB][32];
#pragma unroll
          for (int q = 0; q < T2_GB; ++q) tmem_ld32_nw(taddr + min(b0 + q, nbk - 1) * 32, v[q]);
          tmem_wait();
          if (b0 + T2_GB >= nbk) {  // the chunk's last group: buffer back to the MMA
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mb_arrive(&sm.acc_empty[buf]);
          }
          if (a.mode == 1) continue;
          // block maxima (FMNMX3 trees), ONE threshold for the group:
          // lo = max(running max, the group's maxima) - band <= M - band
          float bmq[T2_GB];
#pragma unroll
          for (int q = 0; q < T2_GB; ++q) {
            const float* x = v[q];
            float t1[11];
#pragma unroll
            for (int y = 0; y < 10; ++y) t1[y] = max3f(x[3 * y], x[3 * y + 1], x[3 * y + 2]);
            t1[10] = fmaxf(x[30], x[31]);
            const float t2a = max3f(t1[0], t1[1], t1[2]), t2b = max3f(t1[3], t1[4], t1[5]);
            const float t2c = max3f(t1[6], t1[7], t1[8]), t2d = fmaxf(t1[9], t1[10]);
            bmq[q] = fmaxf(max3f(t2a, t2b, t2c), t2d);
          }
          float mall = e0s;
#pragma unroll
          for (int q = 0; q < T2_GB; ++q) mall = fmaxf(mall, bmq[q]);
          const float lo = mall - band;
          uint32_t inq[T2_GB];
#pragma unroll
          for (int q = 0; q < T2_GB; ++q) {
            // a block no row of the warp has in band needs no mask (warp-
            // uniform: pays off when the warp's rows share their clusters)
            inq[q] = 0u;
            if (__any_sync(0xffffffffu, bmq[q] >= lo)) inq[q] = ~below_mask32(v[q], lo);
            if (b0 + q >= nbk) inq[q] = 0u;
          }
          // branch-free pair update per block: entry {bm, first column, mask}
#pragma unroll
          for (int q = 0; q < T2_GB; ++q) {
            const float bm = bmq[q];
            const uint32_t in = inq[q], col = cbeg + cc + (b0 + q) * 32;
            // e2, e3 keep no score: e1s bounds them (they were <= e1 when
            // they arrived or were pushed down, and e1s only grows); the
            // entry leaving e3 records that bound in dmax
            const bool p = in != 0u, gt1 = p && bm > e1s, gt0 = p && bm > e0s;
#if CKV_T2_ENTRIES == 4
            dmax = (p && e3m) ? fmaxf(dmax, e1s) : dmax;
            e3c = p ? e2c : e3c;
            e3m = p ? e2m : e3m;
            e2c = p ? (gt1 ? e1c : col) : e2c;
            e2m = p ? (gt1 ? e1m : in) : e2m;
#else
            dmax = p ? fmaxf(dmax, gt1 ? e1s : bm) : dmax;
#endif
            e1s = gt0 ? e0s : (gt1 ? bm : e1s);
            e1c = gt0 ? e0c : (gt1 ? col : e1c);
            e1m = gt0 ? e0m : (gt1 ? in : e1m);
            e0s = gt0 ? bm : e0s;
            e0c = gt0 ? col : e0c;
            e0m = gt0 ? in : e0m;
          }
          // entries that fell below the running max - band can never be
          // candidates (lo <= M - band): e1 and what it bounds are dropped
          if (e1s < lo) { e1s = -INFINITY; e1m = 0u; e2m = 0u; e3m = 0u; }
        }
      }
      // the row's decision: M = e0s; candidates = entries with score >= M - band
      if (row < a.n && a.mode == 0) {
        const float M = e0s, lo = M - band;
        // e1, e2, e3 survive with e1 (their common bound)
        const bool u1 = e1s >= lo;
        bool full = !(M > -INFINITY) || dmax >= lo;
        const uint32_t nin =
            __popc(e0m) + (u1 ? __popc(e1m) + __popc(e2m) + __popc(e3m) : 0u);
        if (e0c + 32 - __ffs(e0m) >= a.C) full = true;  // a padding column survived
        if (u1 && e1c + 32 - __ffs(e1m) >= a.C) full = true;
        if (u1 && e2m && e2c + 32 - __ffs(e2m) >= a.C) full = true;
        if (u1 && e3m && e3c + 32 - __ffs(e3m) >= a.C) full = true;
        auto emit = [&](auto&& put) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (e >= 1 && !u1) break;
            uint32_t m = e == 0 ? e0m : e == 1 ? e1m : e == 2 ? e2m : e3m;
            const uint32_t c = e == 0 ? e0c : e == 1 ? e1c : e == 2 ? e2c : e3c;
            while (m) {
              const uint32_t jj = __clz(m);
              m &= ~(0x80000000u >> jj);
              put(c + jj);
            }
          }
        };
        if (summary) {
          if (nin > 4u) full = true;
          uint32_t i01 = 0u, i23 = 0u, k2 = 0;
          if (!full)
            emit([&](uint32_t c) {
              if (k2 == 0) i01 |= c; else if (k2 == 1) i01 |= c << 16;
              else if (k2 == 2) i23 |= c; else i23 |= c << 16;
              ++k2;
            });
          a.summ[(size_t(unit) * a.n + row) * a.n_slots + range] =
              make_float4(M, __uint_as_float(full ? TC_FULL : nin), __uint_as_float(i01),
                          __uint_as_float(i23));
        } else {
          int32_t* lab = a.labels + size_t(unit) * a.label_stride + row;
          if (nin > uint32_t(TC_NCAND)) full = true;
          if (!full && nin == 1) {
            *lab = int32_t(e0c + __clz(e0m));
          } else {
            *lab = -1;
            const uint32_t slot = w0 * TC_M + atomicAdd(&sm.fix_n, 1u);
            if (slot < a.fix_cap) {
              a.fix_list[slot] = make_uint4(unit, row, full ? TC_FULL : nin, 0u);
              if (!full) {
                uint32_t* fi = a.fix_ids + size_t(slot) * TC_NCAND;
                uint32_t k2 = 0;
                emit([&](uint32_t c) { fi[k2++] = c; });
              }
            }
          }
        }
      }
      next_work(k);
      next_work(k);
    }
  }
#ifdef CKV_T2_PROF
  if (lane == 0) {
    if (wid >= 2) acc_[7] += clock64() - tk0_;
    if (t == 0) acc_[6] += clock64() - tk0_;
    for (int x = 0; x < 8; ++x) if (acc_[x]) atomicAdd(&g_t2prof[x], acc_[x]);
  }
#endif
  __syncthreads();
  if (t == 0) a.fix_count[blockIdx.x] = sm.fix_n;
  if (wid == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// exact re-score of the fix-up keys (clustering.hpp:104-115: argmax of
// dot_f64(key, dir_c), strict >, so ties go to the lowest id).
// One warp per key; lane L holds dims 4L..4L+3.  Every candidate's score is
// computed in f64 with a lane-tree sum (all products are exact in f64; the
// result differs from the sequential chain by < 2^-46 |k|).  If the best two
// are closer than 2^-40 |k|, the order could depend on the chain's rounding,
// so those candidates are re-scored with the sequential chain itself (lane 0).
// A FULL key (more in-band columns than the epilogue kept) scans all C.
__device__ __forceinline__ double exact_dot(const uint16_t* __restrict__ kr,
                                            const float* __restrict__ dc) {
  double s = 0.0;
  const uint4* k4 = reinterpret_cast<const uint4*>(kr);
  const float4* d4 = reinterpret_cast<const float4*>(dc);
#pragma unroll 4
  for (int b = 0; b < D / 8; ++b) {
    const uint4 kk = __ldg(k4 + b);
    const float4 x = __ldg(d4 + 2 * b), y = __ldg(d4 + 2 * b + 1);
    s = __fma_rn(double(__uint_as_float(kk.x << 16)), double(x.x), s);
    s = __fma_rn(double(__uint_as_float(kk.x & 0xffff0000u)), double(x.y), s);
    s = __fma_rn(double(__uint_as_float(kk.y << 16)), double(x.z), s);
    s = __fma_rn(double(__uint_as_float(kk.y & 0xffff0000u)), double(x.w), s);
    s = __fma_rn(double(__uint_as_float(kk.z << 16)), double(y.x), s);
    s = __fma_rn(double(__uint_as_float(kk.z & 0xffff0000u)), double(y.y), s);
    s = __fma_rn(double(__uint_as_float(kk.w << 16)), double(y.z), s);
    s = __fma_rn(double(__uint_as_float(kk.w & 0xffff0000u)), double(y.w), s);
  }
  return s;
}

__device__ __forceinline__ double lane_partial(const double k[4], const float4 d) {
  return __fma_rn(k[3], double(d.w),
                  __fma_rn(k[2], double(d.z), __fma_rn(k[1], double(d.y), k[0] * double(d.x))));
}

__global__ void __launch_bounds__(256)
k_fixup(const uint4* __restrict__ list, const uint32_t* __restrict__ ids,
        const uint32_t* __restrict__ count, const int32_t* __restrict__ n_active,
        uint32_t tiles_per_unit, const uint16_t* __restrict__ keys,
        uint64_t key_stride, const float* __restrict__ dirs, uint32_t C, uint32_t c_pad,
        const float* __restrict__ knorm, uint32_t n, int32_t* __restrict__ labels,
        uint32_t label_stride, uint32_t* __restrict__ full_q = nullptr,
        uint32_t* __restrict__ full_n = nullptr) {
  // region r = blockIdx.y holds count[r] entries from index r * per * 128
  // (k_assign_tc's CTA r processed tiles [r * per, (r + 1) * per)).
  // A half-warp per key (lane hl holds dims 8hl..8hl+7): two keys per warp,
  // 4 shuffle levels per candidate instead of 5 over a whole warp.
  const uint32_t r = blockIdx.y;
  const uint32_t total = uint32_t(*n_active) * tiles_per_unit;
  const uint32_t per = (total + gridDim.y - 1) / gridDim.y;
  const uint32_t nfix = count[r];
  const uint32_t rbase = r * per * TC_M;
  const int lane = lane_id(), hl = lane & 15;
  const unsigned hmask = (lane < 16) ? 0x0000ffffu : 0xffff0000u;
  const uint32_t nh = gridDim.x * (blockDim.x >> 4);  // half-warps in the grid
  for (uint32_t e0 = (blockIdx.x * (blockDim.x >> 5) + warp_id()) * 2 + (lane >> 4); e0 < nfix;
       e0 += nh) {
    const uint32_t e = rbase + e0;
    const uint4 it = list[e];
    const uint32_t u = it.x, row = it.y;
    const bool full = it.z == TC_FULL;
    if (full && full_q) {  // all C columns: a whole CTA per key, k_fixup_full
      if (hl == 0) full_q[atomicAdd(full_n, 1u)] = e;
      continue;
    }
    const uint32_t nc = full ? C : it.z;
    const uint16_t* kr = keys + u * key_stride + size_t(row) * D;
    const uint4 kv = __ldg(reinterpret_cast<const uint4*>(kr) + hl);
    const double k[8] = {double(__uint_as_float(kv.x << 16)), double(__uint_as_float(kv.x & 0xffff0000u)),
                         double(__uint_as_float(kv.y << 16)), double(__uint_as_float(kv.y & 0xffff0000u)),
                         double(__uint_as_float(kv.z << 16)), double(__uint_as_float(kv.z & 0xffff0000u)),
                         double(__uint_as_float(kv.w << 16)), double(__uint_as_float(kv.w & 0xffff0000u))};
    const float* du = dirs + size_t(u) * c_pad * D;
    const uint32_t* cid = ids + size_t(e) * TC_NCAND;
    double best = -INFINITY, second = -INFINITY;
    uint32_t bid = 0xffffffffu;
    for (uint32_t j0 = 0; j0 < nc; j0 += TC_NCAND) {
      double p[TC_NCAND];
      uint32_t c[TC_NCAND];
#pragma unroll
      for (int j = 0; j < TC_NCAND; ++j) {  // 8 independent row loads + partials
        c[j] = j0 + j < nc ? (full ? j0 + j : __ldg(cid + j0 + j)) : 0u;
        const float4* dr = reinterpret_cast<const float4*>(du + size_t(c[j]) * D) + 2 * hl;
        const float4 x = __ldg(dr), y = __ldg(dr + 1);
        p[j] = __fma_rn(k[7], double(y.w), __fma_rn(k[6], double(y.z),
               __fma_rn(k[5], double(y.y), __fma_rn(k[4], double(y.x),
               __fma_rn(k[3], double(x.w), __fma_rn(k[2], double(x.z),
               __fma_rn(k[1], double(x.y), k[0] * double(x.x))))))));
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1)
#pragma unroll
        for (int j = 0; j < TC_NCAND; ++j) p[j] += __shfl_xor_sync(hmask, p[j], o);
#pragma unroll
      for (int j = 0; j < TC_NCAND; ++j) {
        if (j0 + j >= nc) break;
        const double sj = isnan(p[j]) ? -INFINITY : p[j];
        if (sj > best) { second = best; best = sj; bid = c[j]; }  // ids ascend: first max
        else if (sj > second) second = sj;
      }
    }
    const double kn = double(knorm[size_t(u) * n + row]);
    const double tie = kn * 0x1p-40;
    if (!(best - second > tie) && best > -INFINITY) {
      // near-tie: the sequential chain (dot_f64's exact rounding) decides;
      // lanes split the candidates, first maximum per lane, then lowest id
      double b2 = -INFINITY;
      uint32_t i2 = 0xffffffffu;
      for (uint32_t j = hl; j < nc; j += 16) {
        const uint32_t cj = full ? j : cid[j];
        const double sj = exact_dot(kr, du + size_t(cj) * D);
        if (sj > b2) { b2 = sj; i2 = cj; }
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        const double os = __shfl_xor_sync(hmask, b2, o);
        const uint32_t oi = __shfl_xor_sync(hmask, i2, o);
        if (os > b2 || (os == b2 && oi < i2)) { b2 = os; i2 = oi; }
      }
      bid = i2;
    }
    if (hl == 0)
      labels[size_t(u) * label_stride + row] = int32_t(bid == 0xffffffffu ? 0 : bid);
  }
}

// FULL fix-ups (more in-band columns than the epilogue kept: near-ties among
// many centroids): the argmax over all C columns of one key by a whole CTA.
// Warp w takes columns w, w + 8, ...; lane L holds dims 4L..4L+3, the score
// is a lane-tree f64 sum (products exact in f64; within 2^-46 |k| of the
// sequential chain), kept in smem.  When the best two are closer than
// 2^-40 |k|, every column within that of the best is re-scored with the
// sequential dot_f64 chain (the reference's rounding) and the first maximum
// wins (clustering.hpp:104-115).  One launch over the queue k_fixup filled.
constexpr int FF_WARPS = 8;
constexpr uint32_t FF_MAXC = TC_MAXC_ALL;
#ifndef CKV_FF_ROWS
#define CKV_FF_ROWS 16
#endif
constexpr int FF_ROWS = CKV_FF_ROWS;  // centroid rows in flight per warp (k_fixup_full)
__global__ void __launch_bounds__(FF_WARPS * 32)
k_fixup_full(const uint4* __restrict__ list, const uint32_t* __restrict__ full_q,
             const uint32_t* __restrict__ full_n, const uint16_t* __restrict__ keys,
             uint64_t key_stride, const float* __restrict__ dirs, uint32_t C, uint32_t c_pad,
             const float* __restrict__ knorm, uint32_t n, int32_t* __restrict__ labels,
             uint32_t label_stride) {
  __shared__ double sc[FF_MAXC];
  __shared__ double wb[FF_WARPS], ws[FF_WARPS];
  __shared__ uint32_t wi[FF_WARPS];
  __shared__ double s_thr;
  __shared__ uint32_t s_bid, s_tie;
  const int lane = lane_id(), w = warp_id();
  const uint32_t nf = *full_n;
  for (uint32_t qi = blockIdx.x; qi < nf; qi += gridDim.x) {
    const uint4 it = list[full_q[qi]];
    const uint32_t u = it.x, row = it.y;
    const uint16_t* kr = keys + u * key_stride + size_t(row) * D;
    const uint2 kv = __ldg(reinterpret_cast<const uint2*>(kr) + lane);
    const double k0 = double(__uint_as_float(kv.x << 16)), k1 = double(__uint_as_float(kv.x & 0xffff0000u));
    const double k2 = double(__uint_as_float(kv.y << 16)), k3 = double(__uint_as_float(kv.y & 0xffff0000u));
    const float* du = dirs + size_t(u) * c_pad * D;
    double best = -INFINITY, second = -INFINITY;
    uint32_t bid = 0xffffffffu;
    for (uint32_t c0 = w; c0 < C; c0 += FF_WARPS * FF_ROWS) {
      double p[FF_ROWS];
      uint32_t cc[FF_ROWS];
#pragma unroll
      for (int j = 0; j < FF_ROWS; ++j) {  // FF_ROWS rows in flight per warp
        cc[j] = c0 + FF_WARPS * j;
        const float4 x = cc[j] < C ? __ldg(reinterpret_cast<const float4*>(du + size_t(cc[j]) * D) + lane)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
        p[j] = __fma_rn(k3, double(x.w), __fma_rn(k2, double(x.z), __fma_rn(k1, double(x.y), k0 * double(x.x))));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int j = 0; j < FF_ROWS; ++j) p[j] += __shfl_xor_sync(0xffffffffu, p[j], o);
#pragma unroll
      for (int j = 0; j < FF_ROWS; ++j) {
        if (cc[j] >= C) break;
        const double sj = isnan(p[j]) ? -INFINITY : p[j];
        if (lane == 0) sc[cc[j]] = sj;
        if (sj > best) { second = best; best = sj; bid = cc[j]; }  // ids ascend per warp
        else if (sj > second) second = sj;
      }
    }
    if (lane == 0) { wb[w] = best; ws[w] = second; wi[w] = bid; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = -INFINITY, s2 = -INFINITY;
      uint32_t bi = 0xffffffffu;
      for (int x = 0; x < FF_WARPS; ++x) {
        if (wb[x] > b || (wb[x] == b && wi[x] < bi)) { s2 = fmax(s2, b); b = wb[x]; bi = wi[x]; }
        else s2 = fmax(s2, wb[x]);
        s2 = fmax(s2, ws[x]);
      }
      const double tie = double(knorm[size_t(u) * n + row]) * 0x1p-40;
      s_bid = bi;
      s_tie = (b > -INFINITY && !(b - s2 > tie)) ? 1u : 0u;
      s_thr = b - tie;  // the near-tie re-score threshold
    }
    __syncthreads();
    uint32_t label = s_bid;
    if (s_tie) {
      // near-tie: the sequential chain decides among the columns within
      // the tie margin of the best, first maximum (lowest id on equality)
      const double thr = s_thr;
      double b2 = -INFINITY;
      uint32_t i2 = 0xffffffffu;
      for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
        if (!(sc[c] >= thr)) continue;
        const double sj = exact_dot(kr, du + size_t(c) * D);
        if (sj > b2) { b2 = sj; i2 = c; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, b2, o);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, i2, o);
        if (os > b2 || (os == b2 && oi < i2)) { b2 = os; i2 = oi; }
      }
      __syncthreads();
      if (lane == 0) { wb[w] = b2; wi[w] = i2; }
      __syncthreads();
      if (threadIdx.x == 0) {
        double b = -INFINITY;
        uint32_t bi = 0xffffffffu;
        for (int x = 0; x < FF_WARPS; ++x)
          if (wb[x] > b || (wb[x] == b && wi[x] < bi)) { b = wb[x]; bi = wi[x]; }
        s_bid = bi;
      }
      __syncthreads();
      label = s_bid;
    }
    if (threadIdx.x == 0)
      labels[size_t(u) * label_stride + row] = int32_t(label == 0xffffffffu ? 0 : label);
    __syncthreads();  // smem reused by the next key
  }
}

__global__ void k_eps_max(const float* __restrict__ deps, uint32_t c_pad, uint32_t n_units,
                          float* __restrict__ eps_u) {
  const uint32_t u = blockIdx.x * (blockDim.x >> 5) + warp_id();
  if (u >= n_units) return;
  float m = 0.f;
  for (uint32_t c = lane_id(); c < c_pad; c += 32) m = fmaxf(m, deps[size_t(u) * c_pad + c]);
  m = warp_max(m);
  if (lane_id() == 0) eps_u[u] = m;
}

// C > 512: combine a key's per-range summaries (k_assign_tc, n_ranges > 1).
// M = max_r M_r; a range with M_r < M - band holds no candidate; the others
// contribute their in-band ids (each a superset of that range's share of
// {c : S_c >= M - band}).  One candidate -> the label; otherwise the key goes
// to the fix-up list (one region, warp-aggregated slots) with its <= 8
// candidates, or FULL.
__global__ void __launch_bounds__(256)
k_assign_merge(const float4* __restrict__ summ, uint32_t n_ranges, uint32_t n,
               const int32_t* __restrict__ unit_list, const int32_t* __restrict__ n_list,
               const float* __restrict__ knorm, const float* __restrict__ eps_u,
               const float* __restrict__ kerr_u,
               int32_t* __restrict__ labels, uint32_t label_stride, uint4* __restrict__ fix_list,
               uint32_t* __restrict__ fix_ids, uint32_t* __restrict__ fix_n, uint32_t fix_cap) {
  const uint32_t ui = blockIdx.y;
  if (ui >= uint32_t(*n_list)) return;
  const uint32_t unit = uint32_t(unit_list[ui]);
  const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
  bool need = false, full = false;
  uint32_t nin = 0, ids[TC_NCAND];
  if (row < n) {
    const float4* sp = summ + (size_t(unit) * n + row) * n_ranges;
    const float band = tc_band(knorm[size_t(unit) * n + row], eps_u[unit], kerr_u[unit]);
    float M = -INFINITY;
    for (uint32_t r = 0; r < n_ranges; ++r) M = fmaxf(M, sp[r].x);
    full = !(M > -INFINITY);
    for (uint32_t r = 0; r < n_ranges && !full; ++r) {
      const float4 sr = sp[r];
      if (!(sr.x >= M - band)) continue;
      const uint32_t nr = __float_as_uint(sr.y);
      if (nr == TC_FULL || nin + nr > uint32_t(TC_NCAND)) { full = true; break; }
      const uint32_t pk[2] = {__float_as_uint(sr.z), __float_as_uint(sr.w)};
      for (uint32_t k = 0; k < nr; ++k) ids[nin++] = (pk[k >> 1] >> (16 * (k & 1))) & 0xffffu;
    }
    int32_t* lab = labels + size_t(unit) * label_stride + row;
    if (!full && nin == 1) *lab = int32_t(ids[0]);
    else { *lab = -1; need = true; }
  }
  const unsigned m = __ballot_sync(0xffffffffu, need);
  if (!m) return;
  uint32_t base = 0;
  if (lane_id() == 0) base = atomicAdd(fix_n, uint32_t(__popc(m)));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (need) {
    const uint32_t slot = base + __popc(m & ((1u << lane_id()) - 1u));
    if (slot < fix_cap) {
      fix_list[slot] = make_uint4(unit, row, full ? TC_FULL : nin, 0u);
      if (!full)
        for (uint32_t k = 0; k < nin; ++k) fix_ids[size_t(slot) * TC_NCAND + k] = ids[k];
    }
  }
}

// cluster-major fp16 operand: dst row r of a unit = src row sorted[r] (the
// index of the latest labels, so a 128-key tile holds a few clusters and the
// epilogue's warp-uniform block skip applies); rows >= n stay zero and map to
// themselves.  perm[r] = the key position (ckv_kmeans.cu, once per k-means run)
__global__ void __launch_bounds__(256)
k_permute_keys(const uint16_t* __restrict__ k16, uint32_t n, uint32_t n_pad,
               const uint32_t* __restrict__ sorted, uint32_t label_stride,
               const int32_t* __restrict__ active, uint16_t* __restrict__ k16p,
               uint32_t* __restrict__ perm) {
  const uint32_t u = blockIdx.y;
  if (active && !active[u]) return;
  const uint32_t r = blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4);
  if (r >= n_pad) return;
  const uint32_t src = r < n ? sorted[size_t(u) * label_stride + r] : r;
  const uint4* s4 = reinterpret_cast<const uint4*>(k16 + (size_t(u) * n_pad + src) * D);
  uint4* d4 = reinterpret_cast<uint4*>(k16p + (size_t(u) * n_pad + r) * D);
  const int j = threadIdx.x & 15;
  d4[j] = r < n ? s4[j] : make_uint4(0u, 0u, 0u, 0u);
  if (j == 0) perm[size_t(u) * n_pad + r] = src;
}

int launch_permute_keys(cudaStream_t st, const uint16_t* k16, uint32_t n, uint32_t n_pad,
                        const uint32_t* sorted, uint32_t label_stride, uint32_t n_units,
                        const int32_t* active, uint16_t* k16p, uint32_t* perm) {
  k_permute_keys<<<dim3((n_pad + 15) / 16, n_units), 256, 0, st>>>(k16, n, n_pad, sorted,
                                                                    label_stride, active, k16p, perm);
  CKV_LAUNCH_CHECK("k_permute_keys");
  return CKV_OK;
}

__global__ void k_compact_active(const int32_t* __restrict__ active, uint32_t n_units,
                                  int32_t* __restrict__ list, int32_t* __restrict__ count,
                                  uint32_t* __restrict__ fix_count) {
  // one warp: ballots keep the list in ascending unit order
  if (blockIdx.x != 0) return;
  const uint32_t lane = threadIdx.x & 31u;
  if (threadIdx.x >= 32) return;
  uint32_t n = 0;
  for (uint32_t u0 = 0; u0 < n_units; u0 += 32) {
    const uint32_t u = u0 + lane;
    const bool on = u < n_units && (!active || active[u]);
    const unsigned m = __ballot_sync(0xffffffffu, on);
    if (on) list[n + __popc(m & ((1u << lane) - 1u))] = int32_t(u);
    n += __popc(m);
  }
  if (lane == 0) {
    *count = int32_t(n);
    *fix_count = 0;
    fix_count[TC_MERGE_SLOT] = 0;  // k_assign_merge's single region
    fix_count[TC_FULL_SLOT] = 0;   // k_fixup_full's queue length
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
bool assign_tc_supported(uint32_t n, uint32_t C) {
  const uint32_t c_pad = (C + 31) / 32 * 32;
  return C >= 32 && c_pad <= uint32_t(TC_MAXC_ALL) && n >= uint32_t(TC_M);
}

namespace {
struct TcScratch {
  int32_t* list;
  int32_t* count;
  uint32_t* fix_count;
  uint4* fix_list;
  uint32_t* fix_ids;
  uint32_t* full_q;  // FULL fix-up entries, k_fixup -> k_fixup_full
  float* knorm;
  float* eps_u;
  float* kerr;     // [unit] max_k |k - h(k)| (float bits, atomicMax'd as u32)
  uint16_t* k16;   // [unit][n_pad][128] the fp16 tensor-core copy of the keys
  uint32_t n_pad;
  float4* summ;  // C > 512 only: per-(key, range) summaries
  uint32_t fix_cap;
};
// column ranges of <= TC_MAXC columns, balanced, multiples of 32
void tc_ranges(uint32_t c_pad, uint32_t* n_ranges, uint32_t* rc) {
  const uint32_t nr = (c_pad + TC_MAXC - 1) / TC_MAXC;
  *n_ranges = nr;
  *rc = ((c_pad + nr - 1) / nr + 31) / 32 * 32;
}
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
TcScratch carve(void* base, uint32_t n_units, uint32_t n) {
  TcScratch s;
  uint8_t* p = static_cast<uint8_t*>(base);
  s.list = reinterpret_cast<int32_t*>(p);
  p += align256(size_t(n_units) * 4);
  s.count = reinterpret_cast<int32_t*>(p);
  p += 256;
  s.fix_count = reinterpret_cast<uint32_t*>(p);  // [grid] per-CTA counts
  p += 4096;
  s.fix_cap = n_units * ((n + TC_M - 1) / TC_M) * TC_M;  // every key can need a fix-up
  s.fix_list = reinterpret_cast<uint4*>(p);
  p += align256(size_t(s.fix_cap) * 16);
  s.fix_ids = reinterpret_cast<uint32_t*>(p);
  p += align256(size_t(s.fix_cap) * 32);
  s.full_q = reinterpret_cast<uint32_t*>(p);
  p += align256(size_t(s.fix_cap) * 4);
  s.knorm = reinterpret_cast<float*>(p);
  p += align256(size_t(n_units) * n * 4);
  s.eps_u = reinterpret_cast<float*>(p);
  p += align256(size_t(n_units) * 4) + 256;
  s.kerr = reinterpret_cast<float*>(p);
  p += align256(size_t(n_units) * 4);
  s.n_pad = (n + TC_M - 1) / TC_M * TC_M;
  s.k16 = reinterpret_cast<uint16_t*>(p);
  p += align256(size_t(n_units) * s.n_pad * D * 2);
  s.summ = reinterpret_cast<float4*>(p);  // sized by assign_tc_scratch_bytes
  return s;
}
int encode_2d(CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows) {
  const cuuint64_t dims[2] = {cuuint64_t(D), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(D) * 2};
  const cuuint32_t box[2] = {cuuint32_t(TC_BK), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  // Resolved through the runtime so libckv_b200.so has no link-time libcuda
  // dependency (it must load on hosts without a driver, e.g. the CPU tests).
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<EncodeFn>(fn);
  }();
  if (!encode) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return CKV_ECUDA;
  }
  CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                                      const_cast<void*>(base), dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed");
    return CKV_ECUDA;
  }
  return CKV_OK;
}
}  // namespace

// the tensor-core key operands live in the scratch: k_scan_keys (ckv_kmeans.cu)
// fills the fp16 copy, the band norms and the per-unit conversion error once
// per k-means run (keys never change); kerr must be zeroed before it runs
TcKeyPrep assign_tc_keyprep(void* scratch, uint32_t n_units, uint32_t n) {
  const TcScratch s = carve(scratch, n_units, n);
  return TcKeyPrep{s.knorm, s.k16, s.n_pad, reinterpret_cast<uint32_t*>(s.kerr)};
}

size_t assign_tc_scratch_bytes(uint32_t n_units, uint32_t n, uint32_t C) {
  const size_t cap = size_t(n_units) * ((n + TC_M - 1) / TC_M) * TC_M;
  uint32_t nr = 1, rc = 0;
  tc_ranges((C + 31) / 32 * 32, &nr, &rc);
  const size_t summ = nr > 1 ? size_t(n_units) * n * nr * 16 : 0;
  return align256(size_t(n_units) * 4) + 256 + 4096 + align256(cap * 16) + align256(cap * 32) +
         align256(cap * 4) + align256(size_t(n_units) * n * 4) +
         align256(size_t(n_units) * 4) + 256 + align256(size_t(n_units) * 4) +
         align256(cap * D * 2) + summ;
}

#ifdef CKV_T2_PROF
void t2_prof_dump() {
  unsigned long long h[8];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(h, g_t2prof, sizeof(h));
  fprintf(stderr, "[t2prof] kernel %.3g | prod a_empty %.3g | mma a_full %.3g acc_empty %.3g "
          "b_full %.3g | epilogue acc_full %.3g of lifetime %.3g (cycles, summed over CTAs)\n",
          double(h[6]), double(h[0]), double(h[1]), double(h[2]), double(h[5]), double(h[3]),
          double(h[7]));
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbol(g_t2prof, z, sizeof(z));
}
#endif

// k_assign_tc with as many key-tile stages as fit next to B (rc columns)
static int launch_tc(cudaStream_t st, const CUtensorMap& kmap, const CUtensorMap& dmap,
                     TcArgs& ta) {
  // k_assign_tc2 (barrier-free epilogue) for the dense and range passes;
  // k_assign_tc for the MCR work lists (CKV_TC_V1=1 forces it everywhere)
  static const bool v1 = getenv("CKV_TC_V1") != nullptr;
  const bool use2 = !ta.wlist && !v1;
  const void* fn = use2 ? (const void*)k_assign_tc2 : (const void*)k_assign_tc;
  // opt-in per-CTA smem minus the kernel's static part, per device and kernel
  static size_t max_dyn_dev[2][64];
  int dev = 0;
  CKV_CUDA_TRY(cudaGetDevice(&dev));
  size_t max_dyn = max_dyn_dev[use2][dev & 63];
  if (max_dyn == 0) {
    int optin = 0;
    cudaFuncAttributes fa;
    CKV_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    CKV_CUDA_TRY(cudaFuncGetAttributes(&fa, fn));
    max_dyn = size_t(optin) - fa.sharedSizeBytes;
  }
  CKV_CUDA_TRY(smem_optin(fn, int(max_dyn)));
  max_dyn_dev[use2][dev & 63] = max_dyn;
  static const uint32_t tc_mode = getenv("CKV_TC_MODE") ? uint32_t(atoi(getenv("CKV_TC_MODE"))) : 0u;
  ta.mode = tc_mode;
  const size_t fixed = 1024 + 2 * size_t(ta.rc) * 128;
  ta.stages = uint32_t(std::min<size_t>(4, (max_dyn - fixed) / TC_ABYTES));
  if (ta.stages < 2) {
    set_error("assign_tc: not enough shared memory for two key-tile stages");
    return CKV_EINVAL;
  }
  const size_t smem = fixed + size_t(ta.stages) * TC_ABYTES;
  if (use2) {
    k_assign_tc2<<<num_sms(), T2_THREADS, smem, st>>>(kmap, dmap, ta);
    CKV_LAUNCH_CHECK("k_assign_tc2");
#ifdef CKV_T2_PROF
    t2_prof_dump();
#endif
  } else {
    k_assign_tc<<<num_sms(), TC_THREADS, smem, st>>>(kmap, dmap, ta);
    CKV_LAUNCH_CHECK("k_assign_tc");
  }
  return CKV_OK;
}

int assign_tc(cudaStream_t st, const uint16_t* keys, uint64_t key_stride, uint32_t n,
              uint32_t C, uint32_t c_pad, uint32_t n_units, const uint16_t* dirs16,
              const float* deps, const float* dirs, int32_t* labels, uint32_t label_stride, const int32_t* active,
              void* scratch, size_t scratch_bytes, uint64_t* launches, const uint16_t* k16p,
              const uint32_t* perm) {
  (void)scratch_bytes;
  if (key_stride % D) {
    set_error("assign_tc: key stride must be a whole number of rows");
    return CKV_EINVAL;
  }
  TcScratch s = carve(scratch, n_units, n);
  k_compact_active<<<1, 32, 0, st>>>(active, n_units, s.list, s.count, s.fix_count);
  CKV_LAUNCH_CHECK("k_compact_active");
  k_eps_max<<<(n_units + 7) / 8, 256, 0, st>>>(deps, c_pad, n_units, s.eps_u);
  CKV_LAUNCH_CHECK("k_eps_max");
  // A operand: the fp16 key copy (k_scan_keys), [unit][n_pad][128]; the
  // fix-up keeps scoring the original bf16 keys
  CUtensorMap kmap, dmap;
  const uint32_t rows_per_unit = s.n_pad;
  CKV_TRY(encode_2d(&kmap, k16p ? k16p : s.k16, uint64_t(n_units) * rows_per_unit, TC_M));
  CKV_TRY(encode_2d(&dmap, dirs16, uint64_t(n_units) * c_pad, TC_BOXR));
  TcArgs ta;
  ta.perm = k16p ? perm : nullptr;
  ta.unit_list = s.list;
  ta.n_list = s.count;
  ta.n = n;
  ta.C = C;
  ta.c_pad = c_pad;
  ta.tiles_per_unit = (n + TC_M - 1) / TC_M;
  ta.key_rows_per_unit = rows_per_unit;
  ta.label_stride = label_stride;
  ta.knorm = s.knorm;
  ta.eps_u = s.eps_u;
  ta.kerr_u = s.kerr;
  ta.labels = labels;
  ta.fix_count = s.fix_count;
  ta.fix_list = s.fix_list;
  ta.fix_cap = s.fix_cap;
  ta.fix_ids = s.fix_ids;
  tc_ranges(c_pad, &ta.n_ranges, &ta.rc);
  ta.summ = s.summ;
  ta.n_slots = ta.n_ranges;
  ta.wlist = nullptr;
  ta.n_wlist = nullptr;
  CKV_TRY(launch_tc(st, kmap, dmap, ta));
  if (ta.n_ranges == 1) {
    k_fixup<<<dim3(8, num_sms()), 256, 0, st>>>(s.fix_list, s.fix_ids, s.fix_count, s.count,
                                                 ta.tiles_per_unit, keys, key_stride, dirs, C,
                                                 c_pad, s.knorm, n, labels, label_stride, s.full_q,
                                                 s.fix_count + TC_FULL_SLOT);
    CKV_LAUNCH_CHECK("k_fixup");
    k_fixup_full<<<2 * num_sms(), FF_WARPS * 32, 0, st>>>(s.fix_list, s.full_q,
                                                           s.fix_count + TC_FULL_SLOT, keys,
                                                           key_stride, dirs, C, c_pad, s.knorm, n,
                                                           labels, label_stride);
    CKV_LAUNCH_CHECK("k_fixup_full");
    ++*launches;
  } else {
    k_assign_merge<<<dim3((n + 255) / 256, n_units), 256, 0, st>>>(
        s.summ, ta.n_ranges, n, s.list, s.count, s.knorm, s.eps_u, s.kerr, labels, label_stride,
        s.fix_list, s.fix_ids, s.fix_count + TC_MERGE_SLOT, s.fix_cap);
    CKV_LAUNCH_CHECK("k_assign_merge");
    // one region (gridDim.y = 1) holding the merged list
    k_fixup<<<dim3(8 * num_sms(), 1), 256, 0, st>>>(s.fix_list, s.fix_ids,
                                                     s.fix_count + TC_MERGE_SLOT, s.count,
                                                     ta.tiles_per_unit, keys, key_stride, dirs,
                                                     C, c_pad, s.knorm, n, labels, label_stride,
                                                     s.full_q, s.fix_count + TC_FULL_SLOT);
    CKV_LAUNCH_CHECK("k_fixup");
    k_fixup_full<<<2 * num_sms(), FF_WARPS * 32, 0, st>>>(s.fix_list, s.full_q,
                                                           s.fix_count + TC_FULL_SLOT, keys,
                                                           key_stride, dirs, C, c_pad, s.knorm, n,
                                                           labels, label_stride);
    CKV_LAUNCH_CHECK("k_fixup_full");
    ++*launches;
    ++*launches;
  }
  *launches += 4;
  static const bool dbg = getenv("CKV_DEBUG_KMEANS") != nullptr;
  if (dbg) {
    std::vector<uint32_t> cnts(ta.n_ranges == 1 ? num_sms() : 1);
    cudaMemcpyAsync(cnts.data(), ta.n_ranges == 1 ? s.fix_count : s.fix_count + TC_MERGE_SLOT,
                    4 * cnts.size(), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    uint32_t nfix = 0;
    for (uint32_t c : cnts) nfix += c;
    fprintf(stderr, "[kmeans dbg] assign_tc fix-ups %u of %u keys (%.2f%%)\n", nfix,
            n * n_units, 100.0 * nfix / (double(n) * n_units));
  }
  return CKV_OK;
}


// ===========================================================================
// Moved-cluster reduced assignment (MCR), passes t >= 2 of the k-means.
//
// The update of pass t recomputes only the clusters whose member set changed
// (k_update's dirty flags); every other centroid -- hence its direction and
// fp16 operand -- is bit-identical to the one the previous pass scored.  For a
// key whose current label a did not move, s(i, c) is unchanged for every
// unmoved c, and a was the first maximum over all c last pass; so the new
// first maximum lies in {a} U moved.  Such a key ("R") is scored against the
// moved columns only and compared with its exact f64 score of a.  Keys whose
// own cluster moved ("F") are scored against every column.
//
// Keys are gathered into cluster-major order (the previous labels' index) so
// 128-key tiles are mostly all-F or all-R; a tile with any F key is scored
// fully (exact either way).  Columns are permuted moved-first per unit, so an
// R tile's work is one contiguous column block.  k_assign_tc runs from an
// explicit work list in summary mode; k_mcr_merge decides each key (label, or
// the exact f64 fix-up list).  Per unit: no moved cluster -> labels copied;
// too many F tiles -> the dense path.
// ===========================================================================
constexpr int32_t MCR_OFF = 0, MCR_DENSE = 1, MCR_ON = 2, MCR_COPY = 3;

__global__ void __launch_bounds__(256)
k_mcr_plan(uint32_t n, uint32_t C, uint32_t c_pad, uint32_t c_stride, uint32_t label_stride,
           uint32_t tiles, uint32_t rc, uint32_t n_ranges, const int32_t* __restrict__ active,
           const uint8_t* __restrict__ moved, const int32_t* __restrict__ prev,
           const uint32_t* __restrict__ sorted, uint32_t* __restrict__ cperm,
           uint8_t* __restrict__ tclass, int32_t* __restrict__ mode, uint32_t* __restrict__ cnt,
           uint32_t* __restrict__ mpad_out) {
  extern __shared__ uint32_t pre[];  // [C + 1] moved prefix
  __shared__ uint32_t s_w[8], s_nf;
  const uint32_t u = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (!active[u]) {
    if (tid == 0) { mode[u] = MCR_OFF; cnt[u] = 0; }
    return;
  }
  const uint8_t* mv = moved + size_t(u) * c_stride;
  // exclusive prefix of the moved flags (256-wide chunks)
  uint32_t carry = 0;
  for (uint32_t b = 0; b < C; b += 256) {
    const uint32_t c = b + tid;
    const uint32_t f = c < C ? uint32_t(mv[c] != 0) : 0u;
    uint32_t x = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    uint32_t wp = 0, tot = 0;
    for (int w = 0; w < 8; ++w) { if (w < wid) wp += s_w[w]; tot += s_w[w]; }
    if (c < C) pre[c] = carry + wp + x - f;
    __syncthreads();
    carry += tot;
  }
  if (tid == 0) { pre[C] = carry; s_nf = 0; }
  __syncthreads();
  const uint32_t m = pre[C];
  // moved clusters first (ascending), then the unmoved ones (ascending)
  uint32_t* cp = cperm + size_t(u) * c_pad;
  for (uint32_t c = tid; c < C; c += 256)
    cp[mv[c] ? pre[c] : m + (c - pre[c])] = c;
  // tile classes over the cluster-major order of the previous labels
  const int32_t* pl = prev + size_t(u) * label_stride;
  const uint32_t* so = sorted + size_t(u) * label_stride;
  uint32_t nf = 0;
  for (uint32_t T = tid; T < tiles; T += 256) {
    const uint32_t r0 = T * TC_M, r1 = min(n, r0 + TC_M) - 1;
    const uint32_t lf = uint32_t(pl[so[r0]]), ll = uint32_t(pl[so[r1]]);
    const bool F = pre[ll + 1] > pre[lf];
    tclass[size_t(u) * tiles + T] = F ? 1 : 0;
    nf += F;
  }
  nf = __reduce_add_sync(0xffffffffu, nf);
  if (lane == 0) atomicAdd(&s_nf, nf);
  __syncthreads();
  if (tid == 0) {
    const uint32_t mpad = (m + 31) / 32 * 32;
    const uint32_t r_chunks = (mpad + rc - 1) / rc;
    int32_t md = MCR_ON;
    if (m == 0) md = MCR_COPY;
    else if (10ull * s_nf > 6ull * tiles || mpad * 10 > c_pad * 6) md = MCR_DENSE;
    mode[u] = md;
    mpad_out[u] = mpad;
    cnt[u] = md == MCR_ON ? s_nf * n_ranges + (tiles - s_nf) * r_chunks : 0u;
  }
}

// work list of the ON units (F tiles x every column range, then R tiles x
// the moved columns), the permuted fp16 B operand, the dense-unit mask
__global__ void __launch_bounds__(256)
k_mcr_emit(uint32_t U, uint32_t C, uint32_t c_pad, uint32_t tiles, uint32_t rc,
           uint32_t n_ranges, const int32_t* __restrict__ mode, const uint32_t* __restrict__ cnt,
           const uint32_t* __restrict__ mpad, const uint8_t* __restrict__ tclass,
           const uint32_t* __restrict__ cperm, const uint16_t* __restrict__ dirs16,
           uint16_t* __restrict__ bperm, uint4* __restrict__ wlist, int32_t* __restrict__ n_wlist,
           int32_t* __restrict__ dense_active) {
  __shared__ uint32_t s_off, s_w[8], s_nf;
  const uint32_t u = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) dense_active[u] = mode[u] == MCR_DENSE;
  // offset of this unit's items (and the total, by the last unit)
  uint32_t part = 0, all = 0;
  for (uint32_t v = tid; v < U; v += 256) {
    if (v < u) part += cnt[v];
    all += cnt[v];
  }
  part = __reduce_add_sync(0xffffffffu, part);
  all = __reduce_add_sync(0xffffffffu, all);
  if (tid == 0) { s_off = 0; s_nf = 0; }
  __syncthreads();
  if (lane == 0) { atomicAdd(&s_off, part); if (u == U - 1) atomicAdd(n_wlist, int32_t(all)); }
  __syncthreads();
  if (mode[u] != MCR_ON) return;
  const uint32_t off = s_off;
  // B operand in permuted column order (padding rows zero)
  const uint32_t* cp = cperm + size_t(u) * c_pad;
  for (uint32_t e = tid; e < c_pad * (D / 8); e += 256) {
    const uint32_t j = e / (D / 8), q = e % (D / 8);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (j < C) v = __ldg(reinterpret_cast<const uint4*>(dirs16 + (size_t(u) * c_pad + cp[j]) * D) + q);
    reinterpret_cast<uint4*>(bperm + (size_t(u) * c_pad + j) * D)[q] = v;
  }
  // F tiles (compacted, in order) for each range, then R tiles for the moved block
  const uint8_t* tc = tclass + size_t(u) * tiles;
  const uint32_t m_pad = mpad[u];
  uint32_t nF = 0;
  for (uint32_t T = tid; T < tiles; T += 256) nF += tc[T];
  nF = __reduce_add_sync(0xffffffffu, nF);
  if (lane == 0) atomicAdd(&s_nf, nF);
  __syncthreads();
  nF = s_nf;
  // emission (second pass with the totals known)
  const uint32_t totF = nF;
  const uint32_t r_chunks = (m_pad + rc - 1) / rc;
  uint32_t cF = 0, cR = 0;
  for (uint32_t b = 0; b < tiles; b += 256) {
    const uint32_t T = b + tid;
    const uint32_t f = T < tiles ? tc[T] : 0u, r = T < tiles ? 1u - f : 0u;
    uint32_t xf = f, xr = r;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t yf = __shfl_up_sync(0xffffffffu, xf, o);
      const uint32_t yr = __shfl_up_sync(0xffffffffu, xr, o);
      if (lane >= o) { xf += yf; xr += yr; }
    }
    __shared__ uint32_t s_ef[8], s_er[8];
    if (lane == 31) { s_ef[wid] = xf; s_er[wid] = xr; }
    __syncthreads();
    uint32_t pf = 0, pr = 0, tf = 0, tr = 0;
    for (int w = 0; w < 8; ++w) {
      if (w < wid) { pf += s_ef[w]; pr += s_er[w]; }
      tf += s_ef[w];
      tr += s_er[w];
    }
    __syncthreads();
    const uint32_t iF = cF + pf + xf - f, iR = cR + pr + xr - r;
    cF += tf;
    cR += tr;
    if (T < tiles) {
      if (f) {
        for (uint32_t rg = 0; rg < n_ranges; ++rg)
          wlist[off + rg * totF + iF] =
              make_uint4(u, T, rg * rc, min(rc, c_pad - rg * rc) | (rg << 16));
      } else {
        for (uint32_t k = 0; k < r_chunks; ++k)
          wlist[off + n_ranges * totF + k * (tiles - totF) + iR] =
              make_uint4(u, T, k * rc, min(rc, m_pad - k * rc) | (k << 16));
      }
    }
  }
}

// keys (and their norms) of the ON units in cluster-major order
__global__ void __launch_bounds__(256)
k_mcr_gather(const int32_t* __restrict__ mode, const uint16_t* __restrict__ keys,
             uint64_t key_stride, uint32_t n, uint32_t npad, const uint32_t* __restrict__ sorted,
             uint32_t label_stride, const float* __restrict__ knorm, uint16_t* __restrict__ kperm,
             float* __restrict__ knp) {
  const uint32_t u = blockIdx.y;
  if (mode[u] != MCR_ON) return;
  const uint32_t r = blockIdx.x * 16 + (threadIdx.x >> 4), q = threadIdx.x & 15;
  if (r >= npad) return;
  uint4 v = make_uint4(0, 0, 0, 0);
  uint32_t src = 0;
  if (r < n) {
    src = __ldg(sorted + size_t(u) * label_stride + r);
    v = __ldg(reinterpret_cast<const uint4*>(keys + u * key_stride + size_t(src) * D) + q);
  }
  reinterpret_cast<uint4*>(kperm + (size_t(u) * npad + r) * D)[q] = v;
  if (q == 0 && r < n) knp[size_t(u) * n + r] = __ldg(knorm + size_t(u) * n + src);
}

__global__ void k_mcr_copy(const int32_t* __restrict__ mode, const int32_t* __restrict__ prev,
                           int32_t* __restrict__ cur, uint32_t n, uint32_t label_stride) {
  const uint32_t u = blockIdx.y;
  if (mode[u] != MCR_COPY) return;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    cur[size_t(u) * label_stride + i] = prev[size_t(u) * label_stride + i];
}

// per key of an ON unit (row j of the cluster-major order, position sorted[j])
__global__ void __launch_bounds__(256)
k_mcr_merge(const int32_t* __restrict__ mode, uint32_t n, uint32_t tiles, uint32_t n_ranges,
            uint32_t rc, const uint32_t* __restrict__ mpad, const uint8_t* __restrict__ tclass,
            const float4* __restrict__ summ, uint32_t n_slots, const uint32_t* __restrict__ cperm,
            uint32_t c_pad, const uint32_t* __restrict__ sorted, uint32_t label_stride,
            const int32_t* __restrict__ prev, int32_t* __restrict__ cur,
            const uint16_t* __restrict__ keys, uint64_t key_stride, const float* __restrict__ dirs,
            const float* __restrict__ knp, const float* __restrict__ eps_u,
            const float* __restrict__ kerr_u,
            uint4* __restrict__ fix_list, uint32_t* __restrict__ fix_ids,
            uint32_t* __restrict__ fix_n, uint32_t fix_cap) {
  const uint32_t u = blockIdx.y;
  if (mode[u] != MCR_ON) return;
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  bool need = false, full = false;
  uint32_t nin = 0, ids[TC_NCAND], pos = 0;
  if (j < n) {
    pos = __ldg(sorted + size_t(u) * label_stride + j);
    const uint32_t a = uint32_t(prev[size_t(u) * label_stride + pos]);
    const float4* sp = summ + (size_t(u) * n + j) * n_slots;
    // err = one score's rigorous bound; band = 2 err (as k_assign_tc's epilogue)
    const float band = tc_band(knp[size_t(u) * n + j], eps_u[u], kerr_u[u]);
    const bool F = tclass[size_t(u) * tiles + j / TC_M] != 0;
    const uint32_t nsl = F ? n_ranges : (mpad[u] + rc - 1) / rc;
    const uint32_t* cp = cperm + size_t(u) * c_pad;
    float M = -INFINITY;
    for (uint32_t r = 0; r < nsl; ++r) M = fmaxf(M, sp[r].x);
    bool any = M > -INFINITY;
    for (uint32_t r = 0; r < nsl && any && !full; ++r) {
      const float4 sr = sp[r];
      if (!(sr.x >= M - band)) continue;
      const uint32_t nr = __float_as_uint(sr.y);
      if (nr == TC_FULL || nin + nr > uint32_t(TC_NCAND)) { full = true; break; }
      const uint32_t pk[2] = {__float_as_uint(sr.z), __float_as_uint(sr.w)};
      for (uint32_t k = 0; k < nr; ++k) ids[nin++] = cp[(pk[k >> 1] >> (16 * (k & 1))) & 0xffffu];
    }
    int32_t lab = -1;
    if (F) {
      full |= !any;
      if (!full && nin == 1) lab = int32_t(ids[0]);
    } else {
      // exact f64 score of the current label (dot_f64's sequential chain)
      const double sa = exact_dot(keys + u * key_stride + size_t(pos) * D,
                                  dirs + (size_t(u) * c_pad + a) * D);
      const double err = 0.5 * double(band);
      if (!any || double(M) + err < sa) {
        lab = int32_t(a);  // every moved score is below s_a; unmoved ones never beat a
      } else if (!full && nin == 1 && sa < double(M) - err) {
        lab = int32_t(ids[0]);  // a is beaten and one moved column is in band
      } else if (!full) {
        if (nin + 1 > uint32_t(TC_NCAND)) full = true;
        else ids[nin++] = a;
      }
    }
    if (lab >= 0) cur[size_t(u) * label_stride + pos] = lab;
    else { cur[size_t(u) * label_stride + pos] = -1; need = true; }
  }
  const unsigned m = __ballot_sync(0xffffffffu, need);
  if (!m) return;
  uint32_t base = 0;
  if (lane_id() == 0) base = atomicAdd(fix_n, uint32_t(__popc(m)));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (need) {
    const uint32_t slot = base + __popc(m & ((1u << lane_id()) - 1u));
    if (slot < fix_cap) {
      // ids ascending is not required: k_fixup takes the first maximum over
      // the exact scores with the lowest id on ties
      fix_list[slot] = make_uint4(u, pos, full ? TC_FULL : nin, 0u);
      if (!full)
        for (uint32_t k = 0; k < nin; ++k) fix_ids[size_t(slot) * TC_NCAND + k] = ids[k];
    }
  }
}

// ---------------------------------------------------------------------------
// host side of MCR
// ---------------------------------------------------------------------------
namespace {
int mcr_alloc(ckv_ctx* ctx, int slot, size_t bytes, void** p) {
  return ctx_scratch(ctx, slot, bytes, false, p);
}
}  // namespace

// Opt-in (CKV_MCR=1): exact, but on config B the per-pass cluster-major key
// gather costs more than the reduced columns save (145 vs 100 ms prefill,
// DESIGN.md §8); kept for the amortised-permutation follow-up.
bool mcr_enabled() {
  static const bool on = getenv("CKV_MCR") != nullptr;
  return on;
}

int assign_mcr(ckv_ctx* ctx, const uint16_t* keys, uint64_t key_stride, uint32_t n, uint32_t C,
               uint32_t c_pad, uint32_t n_units, uint32_t c_stride, const uint16_t* dirs16,
               const float* deps, const float* dirs, const int32_t* prev, int32_t* cur,
               uint32_t label_stride, const int32_t* active, const uint8_t* moved,
               const uint32_t* sorted, void* tc_scratch, size_t tc_bytes) {
  cudaStream_t st = ctx->stream;
  const uint32_t U = n_units, tiles = (n + TC_M - 1) / TC_M, npad = tiles * TC_M;
  uint32_t n_ranges = 1, rc = 0;
  tc_ranges(c_pad, &n_ranges, &rc);
  TcScratch ts = carve(tc_scratch, U, n);  // key norms (positional) live here
  // scratch: small state, permutations, permuted keys, work list + summaries, fix list
  const size_t a256 = 256;
  auto al = [&](size_t x) { return (x + a256 - 1) / a256 * a256; };
  const size_t b_small = al(U * 4) * 4 + al(U * 4) + 512;
  const size_t b_perm = al(size_t(U) * c_pad * 4) + al(size_t(U) * tiles) + al(size_t(U) * c_pad * D * 2);
  const size_t b_keys = al(size_t(U) * npad * D * 2) + al(size_t(U) * n * 4);
  const size_t n_items = size_t(U) * tiles * (n_ranges + 1);
  const size_t b_work = al(n_items * 16) + al(size_t(U) * n * n_ranges * 16);
  const size_t fix_cap = size_t(U) * n;
  const size_t b_fix = al(fix_cap * 16) + al(fix_cap * TC_NCAND * 4);
  void *p_small, *p_perm, *p_keys, *p_work, *p_fix;
  CKV_TRY(mcr_alloc(ctx, 27, b_small, &p_small));
  CKV_TRY(mcr_alloc(ctx, 28, b_perm, &p_perm));
  CKV_TRY(mcr_alloc(ctx, 29, b_keys, &p_keys));
  CKV_TRY(mcr_alloc(ctx, 30, b_work, &p_work));
  CKV_TRY(mcr_alloc(ctx, 31, b_fix, &p_fix));
  uint8_t* q = static_cast<uint8_t*>(p_small);
  int32_t* mode = reinterpret_cast<int32_t*>(q); q += al(U * 4);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(q); q += al(U * 4);
  uint32_t* mpad = reinterpret_cast<uint32_t*>(q); q += al(U * 4);
  int32_t* dense = reinterpret_cast<int32_t*>(q); q += al(U * 4);
  float* eps_u = reinterpret_cast<float*>(q); q += al(U * 4);
  int32_t* n_wlist = reinterpret_cast<int32_t*>(q);
  uint32_t* fix_n = reinterpret_cast<uint32_t*>(q + 64);
  int32_t* n_one = reinterpret_cast<int32_t*>(q + 128);  // n_list for the work-list launch
  q = static_cast<uint8_t*>(p_perm);
  uint32_t* cperm = reinterpret_cast<uint32_t*>(q); q += al(size_t(U) * c_pad * 4);
  uint8_t* tclass = q; q += al(size_t(U) * tiles);
  uint16_t* bperm = reinterpret_cast<uint16_t*>(q);
  q = static_cast<uint8_t*>(p_keys);
  uint16_t* kperm = reinterpret_cast<uint16_t*>(q); q += al(size_t(U) * npad * D * 2);
  float* knp = reinterpret_cast<float*>(q);
  q = static_cast<uint8_t*>(p_work);
  uint4* wlist = reinterpret_cast<uint4*>(q); q += al(n_items * 16);
  float4* summ = reinterpret_cast<float4*>(q);
  q = static_cast<uint8_t*>(p_fix);
  uint4* fix_list = reinterpret_cast<uint4*>(q); q += al(fix_cap * 16);
  uint32_t* fix_ids = reinterpret_cast<uint32_t*>(q);

  CKV_CUDA_TRY(cudaMemsetAsync(n_wlist, 0, 192, st));  // n_wlist, fix_n, n_one
  k_mcr_plan<<<U, 256, (C + 1) * 4, st>>>(n, C, c_pad, c_stride, label_stride, tiles, rc,
                                           n_ranges, active, moved, prev, sorted, cperm, tclass,
                                           mode, cnt, mpad);
  CKV_LAUNCH_CHECK("k_mcr_plan");
  k_mcr_emit<<<U, 256, 0, st>>>(U, C, c_pad, tiles, rc, n_ranges, mode, cnt, mpad, tclass, cperm,
                                dirs16, bperm, wlist, n_wlist, dense);
  CKV_LAUNCH_CHECK("k_mcr_emit");
  k_mcr_copy<<<dim3(8, U), 256, 0, st>>>(mode, prev, cur, n, label_stride);
  CKV_LAUNCH_CHECK("k_mcr_copy");
  k_mcr_gather<<<dim3((npad + 15) / 16, U), 256, 0, st>>>(mode, ts.k16, uint64_t(ts.n_pad) * D, n,
                                                          npad, sorted, label_stride, ts.knorm,
                                                          kperm, knp);
  CKV_LAUNCH_CHECK("k_mcr_gather");
  k_eps_max<<<(U + 7) / 8, 256, 0, st>>>(deps, c_pad, U, eps_u);
  CKV_LAUNCH_CHECK("k_eps_max");
  ctx->launches += 5;
  // the reduced / full tiles of the ON units, from the work list
  CUtensorMap kmap, dmap;
  CKV_TRY(encode_2d(&kmap, kperm, uint64_t(U) * npad, TC_M));
  CKV_TRY(encode_2d(&dmap, bperm, uint64_t(U) * c_pad, TC_BOXR));
  TcArgs ta;
  ta.perm = nullptr;
  ta.unit_list = mode;  // unused with a work list
  ta.n_list = n_one;
  ta.n = n;
  ta.C = C;
  ta.c_pad = c_pad;
  ta.tiles_per_unit = tiles;
  ta.key_rows_per_unit = npad;
  ta.label_stride = label_stride;
  ta.knorm = knp;
  ta.eps_u = eps_u;
  ta.kerr_u = ts.kerr;
  ta.labels = cur;  // not written in summary mode
  ta.fix_count = ts.fix_count;
  ta.fix_list = nullptr;
  ta.fix_cap = 0;
  ta.fix_ids = nullptr;
  ta.n_ranges = n_ranges;
  ta.rc = rc;
  ta.summ = summ;
  ta.n_slots = n_ranges;
  ta.wlist = wlist;
  ta.n_wlist = n_wlist;
  CKV_TRY(launch_tc(st, kmap, dmap, ta));
  k_mcr_merge<<<dim3((n + 255) / 256, U), 256, 0, st>>>(
      mode, n, tiles, n_ranges, rc, mpad, tclass, summ, n_ranges, cperm, c_pad, sorted,
      label_stride, prev, cur, keys, key_stride, dirs, knp, eps_u, ts.kerr, fix_list, fix_ids, fix_n,
      uint32_t(fix_cap));
  CKV_LAUNCH_CHECK("k_mcr_merge");
  k_fixup<<<dim3(8 * num_sms(), 1), 256, 0, st>>>(fix_list, fix_ids, fix_n, n_one, tiles, keys,
                                                   key_stride, dirs, C, c_pad, ts.knorm, n, cur,
                                                   label_stride);
  CKV_LAUNCH_CHECK("k_fixup");
  ctx->launches += 3;
  // the DENSE units through the ordinary path
  CKV_TRY(assign_tc(st, keys, key_stride, n, C, c_pad, U, dirs16, deps, dirs, cur, label_stride,
                    dense, tc_scratch, tc_bytes, &ctx->launches, nullptr, nullptr));
  static const bool dbg = getenv("CKV_DEBUG_KMEANS") != nullptr;
  if (dbg) {
    std::vector<int32_t> md(U);
    int32_t nw = 0;
    uint32_t nfx = 0;
    cudaMemcpyAsync(md.data(), mode, 4 * U, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&nw, n_wlist, 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&nfx, fix_n, 4, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    uint32_t c[4] = {0, 0, 0, 0};
    for (int32_t v : md) c[v]++;
    fprintf(stderr, "[kmeans dbg] MCR units on %u dense %u copy %u off %u | items %d of %u "
            "dense-equivalent | merge fix-ups %u\n", c[MCR_ON], c[MCR_DENSE], c[MCR_COPY],
            c[MCR_OFF], nw, c[MCR_ON] * tiles * n_ranges, nfx);
  }
  return CKV_OK;
}
}  // namespace ckvb
