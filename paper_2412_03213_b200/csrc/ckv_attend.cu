// ckv_attend.cu — K7: sparse decode attention over the gathered KV
// (attention.hpp:20-69 attention_over / approx_attention), split-K
// flash-decode with a log-sum-exp merge.
//
// Persistent, warp-specialised kernel (one CTA per SM slot):
//   work item  = (q head h, slice s): I_T entries [nt*s/S, nt*(s+1)/S).
//   producer   = warp 4, one elected lane.  For each item it stages the q
//                head's run list (I_T as runs of consecutive KV-store rows,
//                ckv_select) in smem, then for each 64-row tile waits for a
//                free ring stage and issues one TMA bulk copy
//                (cp.async.bulk ... mbarrier::complete_tx) per contiguous run
//                segment for K and for V; the stage's mbarrier completes when
//                the bytes land.  The query vector rides a 2-slot ring the
//                same way.  Tiles stream back to back across item
//                boundaries, so the HBM pipeline never drains.
//   consumers  = warps 0-3.  A half-warp owns one row per step (16 lanes x 8
//                bf16 dims): dot product (fp32 FMA + 4 shuffles), online
//                softmax (m, l, acc[8]) per half-warp; each warp releases the
//                stage to the producer.  At the end of an item the 8
//                half-warp states merge in smem into the item partial; the
//                last CTA to finish a q head (atomic ticket) merges its S
//                partials in a fixed order, so results never depend on
//                scheduling.
// Numerics: fp32 logits / exp2 / sums; the reference uses f64 — tolerance-
// checked against the oracle (tests/test_gpu_attend.py).
#include "ckv_internal.cuh"

namespace ckvb {

constexpr int AT_CWARPS = 4;                      // consumer warps
constexpr int AT_THREADS = (AT_CWARPS + 1) * 32;  // + producer warp
#ifndef CKV_AT_TILE
#define CKV_AT_TILE 64
#endif
#ifndef CKV_AT_STAGES
#define CKV_AT_STAGES 2
#endif
constexpr int AT_TILE = CKV_AT_TILE;              // rows per stage (multiple of 8)
constexpr int AT_STAGES = CKV_AT_STAGES;
constexpr int AT_RPH = AT_TILE / 8;               // rows per half-warp per tile
constexpr int AT_RUNS = 256;                      // runs staged in smem
constexpr int PART = 2 + D;                       // partial: m (log2 domain), l, acc[128]

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
// Every consumer thread arrives on a ring slot's empty barrier (count
// AT_CWARPS * 32) instead of one elected lane after __syncwarp: the same
// ordering, but expressed per thread so compute-sanitizer's racecheck can see
// it (it does not treat __syncwarp as ordering a lane's reads before another
// lane's arrive).  Measured: 118.8-119.1 vs 118.4-118.9 us per config B step.
#ifndef CKV_AT_ARRIVE_ALL
#define CKV_AT_ARRIVE_ALL 1
#endif
constexpr uint32_t AT_EMPTY_COUNT = CKV_AT_ARRIVE_ALL ? AT_CWARPS * 32 : AT_CWARPS;
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// the KV rows are read once per step: evict_first, so the stream does not
// push the selection's centroids (evict_last) out of L2
#ifndef CKV_AT_L2HINT
#define CKV_AT_L2HINT 1
#endif
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes,
                                                uint64_t* bar, uint64_t pol) {
  if (!CKV_AT_L2HINT) { bulk_g2s(dst, src, bytes, bar); return; }
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ float ex2(float x) {  // 2^x, ex2.approx (-inf -> +0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(AT_CWARPS * 32) : "memory");
}

#ifndef CKV_AT_FFMA2
#define CKV_AT_FFMA2 1  // packed f32 FMAs (FFMA2) for the logits and the value update
#endif
__device__ __forceinline__ float dot8(const uint4 k, const float* qv) {
#if CKV_AT_FFMA2
  float2 s = make_float2(0.f, 0.f);
  s = __ffma2_rn(make_float2(__uint_as_float(k.x << 16), __uint_as_float(k.x & 0xffff0000u)),
                 make_float2(qv[0], qv[1]), s);
  s = __ffma2_rn(make_float2(__uint_as_float(k.y << 16), __uint_as_float(k.y & 0xffff0000u)),
                 make_float2(qv[2], qv[3]), s);
  s = __ffma2_rn(make_float2(__uint_as_float(k.z << 16), __uint_as_float(k.z & 0xffff0000u)),
                 make_float2(qv[4], qv[5]), s);
  s = __ffma2_rn(make_float2(__uint_as_float(k.w << 16), __uint_as_float(k.w & 0xffff0000u)),
                 make_float2(qv[6], qv[7]), s);
  return s.x + s.y;
#else
  float s = 0.f;
  s = fmaf(__uint_as_float(k.x << 16), qv[0], s);
  s = fmaf(__uint_as_float(k.x & 0xffff0000u), qv[1], s);
  s = fmaf(__uint_as_float(k.y << 16), qv[2], s);
  s = fmaf(__uint_as_float(k.y & 0xffff0000u), qv[3], s);
  s = fmaf(__uint_as_float(k.z << 16), qv[4], s);
  s = fmaf(__uint_as_float(k.z & 0xffff0000u), qv[5], s);
  s = fmaf(__uint_as_float(k.w << 16), qv[6], s);
  s = fmaf(__uint_as_float(k.w & 0xffff0000u), qv[7], s);
  return s;
#endif
}

// acc *= sc in packed pairs
__device__ __forceinline__ void scale8(float sc, float* acc) {
#if CKV_AT_FFMA2
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 r = __fmul2_rn(make_float2(acc[2 * i], acc[2 * i + 1]), make_float2(sc, sc));
    acc[2 * i] = r.x;
    acc[2 * i + 1] = r.y;
  }
#else
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] *= sc;
#endif
}

__device__ __forceinline__ void axpy8(float p, const uint4 v, float* acc) {
#if CKV_AT_FFMA2
  const float2 pp = make_float2(p, p);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 r = __ffma2_rn(
        pp, make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xffff0000u)),
        make_float2(acc[2 * i], acc[2 * i + 1]));
    acc[2 * i] = r.x;
    acc[2 * i + 1] = r.y;
  }
#else
  acc[0] = fmaf(p, __uint_as_float(v.x << 16), acc[0]);
  acc[1] = fmaf(p, __uint_as_float(v.x & 0xffff0000u), acc[1]);
  acc[2] = fmaf(p, __uint_as_float(v.y << 16), acc[2]);
  acc[3] = fmaf(p, __uint_as_float(v.y & 0xffff0000u), acc[3]);
  acc[4] = fmaf(p, __uint_as_float(v.z << 16), acc[4]);
  acc[5] = fmaf(p, __uint_as_float(v.z & 0xffff0000u), acc[5]);
  acc[6] = fmaf(p, __uint_as_float(v.w << 16), acc[6]);
  acc[7] = fmaf(p, __uint_as_float(v.w & 0xffff0000u), acc[7]);
#endif
}

struct __align__(128) AttSmem {
  uint4 k[AT_STAGES][AT_TILE][16];  // AT_TILE x 256 B per stage
  uint4 v[AT_STAGES][AT_TILE][16];
  float q[2][D];                    // query ring
  uint64_t full[AT_STAGES], empty[AT_STAGES], qfull[2], qempty[2];
  uint32_t roff[AT_RUNS + 1], rrow[AT_RUNS];  // producer: runs of the current item
  uint4 item[2];                    // the q slot's work item {i, h, e0, e1} (i = ~0: done)
  float hm[8], hl[8];
  float hacc[8][D];
  uint32_t last;
};

struct ItemInfo {
  uint32_t h, s, e0, e1;
};
// StepSync (ckv_internal.cuh): wait until the selection has published q head
// h for this step.  The acquire makes its run / count stores visible; they
// are then read through L2 (__ldcg), never a possibly stale L1 line.
__device__ __noinline__ void ready_timeout(uint32_t h, uint32_t want) {
  printf("[ckv] k_attend: q head %u never published (want %u)\n", h, want);
  __trap();
}
__device__ __forceinline__ void wait_ready(const uint32_t* ready, uint32_t h, uint32_t want) {
  uint32_t v, n = 0;
  uint64_t t0 = 0;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready + h) : "memory");
    if (v == want) return;
    __nanosleep(64);
    if ((++n & 1023u) == 0u) {  // watchdog: ~4 s
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > 4000000000ull) ready_timeout(h, want);
    }
  }
}
template <bool WEIGHTS>
__global__ void __launch_bounds__(AT_THREADS, 3)
k_attend(ckv_attend_desc desc, uint32_t splits, const float* __restrict__ q,
         const uint16_t* __restrict__ K, const uint16_t* __restrict__ V,
         const uint32_t* __restrict__ rows, ckv_runs runs, const uint32_t* __restrict__ n_tokens,
         float* __restrict__ out, float* __restrict__ logits_ws, float* __restrict__ part,
         uint32_t* __restrict__ tickets, float* __restrict__ weights, float* __restrict__ lse,
         const uint32_t* __restrict__ ready, const uint32_t* __restrict__ epoch,
         uint32_t* __restrict__ work) {
  extern __shared__ __align__(128) unsigned char sm_raw[];
  AttSmem& sm = *reinterpret_cast<AttSmem*>(sm_raw);
  const int t = threadIdx.x, wid = t >> 5, lane = t & 31;
  const uint32_t n_items = desc.n_q * splits;
  if (t == 0) {
    for (int s = 0; s < AT_STAGES; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], AT_EMPTY_COUNT);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.qfull[s], 1);
      mbar_init(&sm.qempty[s], AT_EMPTY_COUNT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // launched with programmatic stream serialization: the CTAs start (and set
  // up their barriers) while the selection kernel drains; its run lists and
  // token counts are read only after this wait (a no-op otherwise).  The next
  // kernel may launch now: it waits for this grid before its dependent reads.
  // StepSync: no grid-wide wait; each item waits for its q head instead (the
  // selection is still running).  Everything else read here was written by
  // kernels that completed before the selection passed its own wait.
  uint32_t want = 0u;
  if (ready) {
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(want) : "l"(epoch) : "memory");
    ++want;
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (wid == AT_CWARPS) {
    // ======================= producer warp =====================================
    uint32_t st = 0, ph = 0, qk = 0;  // ring stage / parity, query-ring counter
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    // the CTA's next item: a fixed stride, or (StepSync) the shared counter,
    // so items are taken in q-head order as the selection publishes them
    uint32_t kf = 0;
    auto fetch = [&]() -> uint32_t {
      uint32_t i = blockIdx.x + (kf++) * gridDim.x;
      if (work) {
        if (lane == 0) i = atomicAdd(work, 1u);
        i = __shfl_sync(0xffffffffu, i, 0);
      }
      return i;
    };
    // An item's metadata (token count, run count, up to AT_RUNS runs) is
    // loaded into registers one item AHEAD, while the current item's tiles
    // stream, so an item start costs no dependent global round trips.  Every
    // lane acquires the head's flag itself before its loads (StepSync).
    constexpr int MO = (AT_RUNS + 1 + 31) / 32, MR = (AT_RUNS + 31) / 32;
    const uint32_t n_off = min(runs.run_cap + 1, uint32_t(AT_RUNS + 1));
    const uint32_t n_row = min(runs.run_cap, uint32_t(AT_RUNS));
    uint32_t m_nt = 0, m_nrun = 0, m_off[MO], m_row[MR];
    auto meta_load = [&](uint32_t i) {
      const uint32_t h = i / splits;
      m_nt = __ldcg(n_tokens + h);
      if (!rows) {
        m_nrun = __ldcg(runs.count + h);
        const uint32_t* gro = runs.off + size_t(h) * (runs.run_cap + 1);
        const uint32_t* grr = runs.row + size_t(h) * runs.run_cap;
#pragma unroll
        for (int k = 0; k < MO; ++k) {
          const uint32_t r = lane + 32 * k;
          m_off[k] = r < n_off ? __ldcg(gro + r) : 0u;
        }
#pragma unroll
        for (int k = 0; k < MR; ++k) {
          const uint32_t r = lane + 32 * k;
          m_row[k] = r < n_row ? __ldcg(grr + r) : 0u;
        }
      }
    };
    auto published = [&](uint32_t i) -> bool {  // non-blocking, per lane
      if (!ready) return true;
      uint32_t v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready + i / splits)
                   : "memory");
      return __all_sync(0xffffffffu, v == want);
    };
    uint32_t i = fetch();
    bool have = false;
    if (i < n_items && published(i)) { meta_load(i); have = true; }
    for (;; ++qk) {
      if (i >= n_items) {  // tell the consumers through the q slot
        if (lane == 0) {
          const uint32_t qs = qk & 1, qp = (qk >> 1) & 1;
          mbar_wait(&sm.qempty[qs], qp ^ 1);
          sm.item[qs] = make_uint4(~0u, 0u, 0u, 0u);
          mbar_arrive(&sm.qfull[qs]);
        }
        break;
      }
      if (!have) {
        if (ready) wait_ready(ready, i / splits, want);
        meta_load(i);
      }
      ItemInfo it;
      it.h = i / splits;
      it.s = i % splits;
      it.e0 = uint32_t((uint64_t(m_nt) * it.s) / splits);
      it.e1 = uint32_t((uint64_t(m_nt) * (it.s + 1)) / splits);
      const uint32_t unit = it.h / desc.group;
      const uint16_t* Ku = K + size_t(unit) * desc.p_cap * D;
      const uint16_t* Vu = V + size_t(unit) * desc.p_cap * D;
      // this item's runs into shared memory (the previous item's issue loop,
      // lane 0 below, is done with them: the warp has reconverged)
      const uint32_t nrun = m_nrun;
      const bool staged = !rows && nrun <= uint32_t(AT_RUNS);
      const uint32_t* gro = rows ? nullptr : runs.off + size_t(it.h) * (runs.run_cap + 1);
      const uint32_t* grr = rows ? nullptr : runs.row + size_t(it.h) * runs.run_cap;
      __syncwarp();
      if (staged) {
#pragma unroll
        for (int k = 0; k < MO; ++k) {
          const uint32_t r = lane + 32 * k;
          if (r <= nrun && r < n_off) sm.roff[r] = m_off[k];
        }
#pragma unroll
        for (int k = 0; k < MR; ++k) {
          const uint32_t r = lane + 32 * k;
          if (r < nrun && r < n_row) sm.rrow[r] = m_row[k];
        }
      }
      __syncwarp();
      // look ahead: the next item and, if its head is published, its metadata
      const uint32_t i_next = fetch();
      have = false;
      if (i_next < n_items && published(i_next)) { meta_load(i_next); have = true; }
      if (lane == 0) {
        const uint32_t qs = qk & 1, qp = (qk >> 1) & 1;
        mbar_wait(&sm.qempty[qs], qp ^ 1);
        sm.item[qs] = make_uint4(i, it.h, it.e0, it.e1);  // released by the arrive below
        mbar_expect_tx(&sm.qfull[qs], D * 4);
        // the selection may have just written q's device copy (zero-copy
        // step): order those generic-proxy stores before this bulk copy
        if (ready) asm volatile("fence.proxy.async.global;" ::: "memory");
        bulk_g2s(sm.q[qs], q + size_t(it.h) * D, D * 4, &sm.qfull[qs]);
        const uint32_t* rowlist = rows ? rows + size_t(it.h) * desc.sel_cap : nullptr;
        uint32_t r = 0;
        if (!rows) {  // last run with off <= e0
          uint32_t lo = 0, hi = nrun;
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if ((staged ? sm.roff[mid] : __ldcg(gro + mid)) <= it.e0) lo = mid; else hi = mid;
          }
          r = lo;
        }
        for (uint32_t e = it.e0; e < it.e1; e += AT_TILE) {
          const uint32_t te = min(e + AT_TILE, it.e1);
          mbar_wait(&sm.empty[st], ph ^ 1);
          mbar_expect_tx(&sm.full[st], (te - e) * D * 2 * 2);
          for (uint32_t x = e; x < te;) {
            uint32_t row, n;
            if (rows) {
              row = __ldg(rowlist + x);
              n = 1;
            } else {
              while ((staged ? sm.roff[r + 1] : __ldcg(gro + r + 1)) <= x) ++r;
              const uint32_t ro = staged ? sm.roff[r] : __ldcg(gro + r);
              const uint32_t rend = staged ? sm.roff[r + 1] : __ldcg(gro + r + 1);
              row = (staged ? sm.rrow[r] : __ldcg(grr + r)) + (x - ro);
              n = min(te, rend) - x;
            }
            bulk_g2s_stream(&sm.k[st][x - e][0], Ku + size_t(row) * D, n * D * 2, &sm.full[st], pol);
            bulk_g2s_stream(&sm.v[st][x - e][0], Vu + size_t(row) * D, n * D * 2, &sm.full[st], pol);
            x += n;
          }
          if (++st == AT_STAGES) { st = 0; ph ^= 1; }
        }
      }
      st = __shfl_sync(0xffffffffu, st, 0);
      ph = __shfl_sync(0xffffffffu, ph, 0);
      i = i_next;
    }
    // StepSync: this grid never completes before the selection grid
    if (ready) asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }

  // ========================= consumer warps ====================================
  const int hw = t >> 4;  // half-warp 0..7
  const int hl = t & 15;  // dims [8*hl, 8*hl+8)
  const float qscale = 1.4426950408889634f * rsqrtf(float(D));  // exp -> exp2
  uint32_t st = 0, ph = 0, qk = 0;
  for (;; ++qk) {
    const uint32_t qs = qk & 1, qp = (qk >> 1) & 1;
    mbar_wait(&sm.qfull[qs], qp);  // the producer's item descriptor and q
    const uint4 d4 = sm.item[qs];
    if (d4.x == ~0u) break;
    const uint32_t i = d4.x;
    ItemInfo it;
    it.h = d4.y;
    it.s = i % splits;
    it.e0 = d4.z;
    it.e1 = d4.w;
    float qv[8];
    {
      const float4 a = *reinterpret_cast<const float4*>(&sm.q[qs][8 * hl]);
      const float4 b = *reinterpret_cast<const float4*>(&sm.q[qs][8 * hl + 4]);
      qv[0] = a.x * qscale; qv[1] = a.y * qscale; qv[2] = a.z * qscale; qv[3] = a.w * qscale;
      qv[4] = b.x * qscale; qv[5] = b.y * qscale; qv[6] = b.z * qscale; qv[7] = b.w * qscale;
    }
    if (CKV_AT_ARRIVE_ALL) {
      mbar_arrive(&sm.qempty[qs]);
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.qempty[qs]);
    }
    float m = -INFINITY, l = 0.f;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float* lw = WEIGHTS ? logits_ws + size_t(it.h) * desc.sel_cap : nullptr;
    for (uint32_t e = it.e0; e < it.e1; e += AT_TILE) {
      mbar_wait(&sm.full[st], ph);
      const bool full_tile = e + AT_TILE <= it.e1;
      float s[AT_RPH];
      uint4 vv[AT_RPH];
#pragma unroll
      for (int kk = 0; kk < AT_RPH; ++kk) {
        const int r = hw + 8 * kk;
        const uint4 kr = sm.k[st][r][hl];
        vv[kk] = sm.v[st][r][hl];
        float x = dot8(kr, qv);
        x += __shfl_xor_sync(0xffffffffu, x, 8);
        x += __shfl_xor_sync(0xffffffffu, x, 4);
        x += __shfl_xor_sync(0xffffffffu, x, 2);
        x += __shfl_xor_sync(0xffffffffu, x, 1);
        s[kk] = x;
      }
      if (CKV_AT_ARRIVE_ALL) {
        mbar_arrive(&sm.empty[st]);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[st]);
      }  // stage data is in registers now
      if (++st == AT_STAGES) { st = 0; ph ^= 1; }
      if (full_tile) {
        if (WEIGHTS && hl == 0)
#pragma unroll
          for (int kk = 0; kk < AT_RPH; ++kk) lw[e + hw + 8 * kk] = s[kk];
        float mn = m;
#pragma unroll
        for (int kk = 0; kk < AT_RPH; ++kk) mn = fmaxf(mn, s[kk]);
        const float sc = ex2(m - mn);  // m = -inf -> 0
        l *= sc;
        scale8(sc, acc);
#pragma unroll
        for (int kk = 0; kk < AT_RPH; ++kk) {
          const float p = ex2(s[kk] - mn);
          l += p;
          axpy8(p, vv[kk], acc);
        }
        m = mn;
      } else {  // the slice's last, partial tile: rows past its end hold stale data
        float tmax = -INFINITY;
#pragma unroll
        for (int kk = 0; kk < AT_RPH; ++kk) {
          const bool ok = e + hw + 8 * kk < it.e1;
          if (WEIGHTS && ok && hl == 0) lw[e + hw + 8 * kk] = s[kk];
          s[kk] = ok ? s[kk] : -INFINITY;
          tmax = fmaxf(tmax, s[kk]);
        }
        const float mn = fmaxf(m, tmax);
        if (mn != -INFINITY) {
          const float sc = ex2(m - mn);
          l *= sc;
          scale8(sc, acc);
#pragma unroll
          for (int kk = 0; kk < AT_RPH; ++kk) {
            if (s[kk] != -INFINITY) {
              const float p = ex2(s[kk] - mn);
              l += p;
              axpy8(p, vv[kk], acc);
            }
          }
          m = mn;
        }
      }
    }
    // ---- merge the 8 half-warp states into the item partial -------------------
    consumer_bar();  // the previous item's merge scratch is free
    if (hl == 0) { sm.hm[hw] = m; sm.hl[hw] = l; }
#pragma unroll
    for (int j = 0; j < 8; ++j) sm.hacc[hw][8 * hl + j] = acc[j];
    consumer_bar();
    float M = sm.hm[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) M = fmaxf(M, sm.hm[j]);
    float* pp = part + size_t(i) * PART;
    {
      float a = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float w = sm.hm[j] == -INFINITY ? 0.f : exp2f(sm.hm[j] - M);
        a += sm.hacc[j][t] * w;
      }
      pp[2 + t] = a;  // 128 consumer threads == D
    }
    if (t == 0) {
      float ls = 0.f;
      for (int j = 0; j < 8; ++j)
        ls += sm.hm[j] == -INFINITY ? 0.f : sm.hl[j] * exp2f(sm.hm[j] - M);
      pp[0] = M;
      pp[1] = ls;
    }
    // ---- the last CTA to finish a q head merges its S partials -----------------
    // bar.sync orders the CTA's partial stores before thread 0's release; the
    // acq_rel RMW makes every other CTA's released partials visible to the
    // last one (PTX release/acquire cumulativity), no per-thread fences.
    consumer_bar();
    if (t == 0) sm.last = (atom_add_acq_rel(&tickets[it.h], 1u) == splits - 1);
    consumer_bar();
    if (sm.last) {
      const float* pb = part + size_t(it.h) * splits * PART;
      float MM = -INFINITY;
      for (uint32_t c = 0; c < splits; ++c) MM = fmaxf(MM, __ldcg(pb + c * PART));
      float L = 0.f, o = 0.f;
      for (uint32_t c = 0; c < splits; ++c) {
        const float mc = __ldcg(pb + c * PART);
        const float w = mc == -INFINITY ? 0.f : exp2f(mc - MM);
        L += __ldcg(pb + c * PART + 1) * w;
        o += __ldcg(pb + c * PART + 2 + t) * w;
      }
      // lse (the sequence-sharded path): this rank's log2-sum-exp2 of the
      // scaled logits beside its locally normalised output; a q head with no
      // local tokens contributes out = 0, lse = -inf to the merge
      const float invL = L > 0.f ? 1.f / L : 0.f;
      out[size_t(it.h) * D + t] = lse && !(L > 0.f) ? 0.f : o * (lse ? invL : 1.f / L);
      if (lse && t == 0) lse[it.h] = L > 0.f ? MM + __log2f(L) : -INFINITY;
      if (WEIGHTS) {
        const uint32_t nt = __ldcg(n_tokens + it.h);
        const float* lg = logits_ws + size_t(it.h) * desc.sel_cap;
        float* wo = weights + size_t(it.h) * desc.sel_cap;
        for (uint32_t j = t; j < nt; j += AT_CWARPS * 32)
          wo[j] = exp2f(__ldcg(lg + j) - MM) * invL;
      }
      if (t == 0) tickets[it.h] = 0;  // re-arm for the next launch
    }
  }
  if (ready) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// work items that fill the GPU twice over at 3 resident CTAs per SM
static uint32_t attend_target_items() {
  static int sms_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int n = sms_dev[dev & 63];
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    n = n < 1 ? 148 : n;
    sms_dev[dev & 63] = n;
  }
  return uint32_t(n) * 6;
}

uint32_t attend_splits(const ckv_attend_desc& d) {
  // ~1024 rows per work item: few per-item epilogues and merges, enough items
  // to balance.  Tile / stage / item sizes were swept on B200 at config B
  // (tools/attend_sweep.sh): 64-row tiles x 2 stages (64 KB ring, 3 CTAs per
  // SM) with 1024-row items gave 94.5 us vs 102 us for 32 x 4 with 512.
#ifndef CKV_AT_ITEM_ROWS
#define CKV_AT_ITEM_ROWS 1024
#endif
  uint32_t s = (d.max_tokens + CKV_AT_ITEM_ROWS - 1) / CKV_AT_ITEM_ROWS;
  // few q heads (one layer's launch in layer mode): split finer, down to
  // 128-row items, so ~2 waves of items cover the SMs (3 CTAs each)
  const uint32_t target = attend_target_items();
  if (d.n_q && uint64_t(d.n_q) * s < target) {
    const uint32_t want = (target + d.n_q - 1) / d.n_q;
    const uint32_t cap = (d.max_tokens + 127) / 128;
    s = std::max(s, std::min(want, cap));
  }
  return s < 1 ? 1 : (s > 64 ? 64 : s);
}

int launch_attend(cudaStream_t st, const ckv_attend_desc& desc, const float* q,
                  const uint16_t* K, const uint16_t* V, const uint32_t* rows,
                  const ckv_runs& runs, const uint32_t* n_tokens, float* out, float* weights,
                  float* logits_ws, float* part, uint32_t* tickets, float* lse,
                  const StepSync* sync) {
  if (!rows && !runs.row) { set_error("attend: need rows or runs"); return CKV_EINVAL; }
  if (desc.n_q == 0 || desc.max_tokens == 0) return CKV_OK;
  const uint32_t splits = attend_splits(desc);
  const size_t smem = sizeof(AttSmem);
  static int per_sm_dev[64];  // resident CTAs per SM, per device (0 = not queried yet)
  int dev = 0;
  CKV_CUDA_TRY(cudaGetDevice(&dev));
  // k_attend<false> always (the occupancy query below uses it)
  CKV_CUDA_TRY(smem_optin((const void*)k_attend<false>, int(smem), true));
  if (weights) CKV_CUDA_TRY(smem_optin((const void*)k_attend<true>, int(smem), true));
  int per_sm = per_sm_dev[dev & 63];
  if (per_sm == 0) {
    CKV_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_attend<false>,
                                                               AT_THREADS, smem));
    per_sm = per_sm < 1 ? 1 : per_sm;
    per_sm_dev[dev & 63] = per_sm;
  }
  const uint32_t n_items = desc.n_q * splits;
  const uint32_t grid = std::min<uint32_t>(n_items, uint32_t(std::max(1, per_sm)) * num_sms());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(AT_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // StepSync only for run lists (the selection publishes per q head)
  const bool use_sync = sync && sync->published && !rows;
  const uint32_t* rdy = use_sync ? sync->ready : nullptr;
  const uint32_t* ep = use_sync ? sync->epoch : nullptr;
  uint32_t* wk = use_sync ? sync->work : nullptr;
  if (weights)
    CKV_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_attend<true>, desc, splits, q, K, V, rows, runs,
                                    n_tokens, out, logits_ws, part, tickets, weights, lse, rdy,
                                    ep, wk));
  else
    CKV_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_attend<false>, desc, splits, q, K, V, rows, runs,
                                    n_tokens, out, static_cast<float*>(nullptr), part, tickets,
                                    static_cast<float*>(nullptr), lse, rdy, ep, wk));
  CKV_LAUNCH_CHECK("k_attend");
  return CKV_OK;
}

size_t attend_part_floats(uint32_t n_q, uint32_t max_tokens) {
  ckv_attend_desc d{};
  d.n_q = n_q;
  d.max_tokens = max_tokens;
  // a launch over any subset of these q heads (layer mode) fits too: it
  // needs <= max(n_q * splits, target + n_q) partials
  return std::max(size_t(n_q) * attend_splits(d), size_t(attend_target_items()) + n_q) * PART;
}

}  // namespace ckvb
