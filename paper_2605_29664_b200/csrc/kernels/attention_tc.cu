// Flash-attention forward on the 5th-generation tensor cores (sm_100a).
//
// Persistent CTAs (one per SM) over (256-query pair tile, head, sequence) tiles, 12 warps:
//   warp 0     : TMA producer — Q_A, Q_B once, then K_j / V_j (128 keys) into 2-stage rings
//                straight out of the packed qkv activation rows;
//   warp 1     : tcgen05.mma issuer, ping-pong order  S_A(j) | PV_B(j-1) | S_B(j) | PV_A(j):
//                while warpgroup A turns S_A(j) into P_A(j) the tensor core runs B's work
//                and vice versa;
//   warp 2     : TMEM allocator (512 columns: S_A | S_B | O_A | O_B);
//   warps 4-7  : softmax warpgroup A (query rows 0-127 of the pair tile);
//   warps 8-11 : softmax warpgroup B (rows 128-255).
// Each K/V tile feeds 256 queries, halving the K/V traffic of a 128-query CTA (the K/V
// stream was the bottleneck: profiles/r01_attn_traces.md).  P never touches smem: the
// softmax threads write it (bf16) over the first 64 TMEM columns of the S tile they just
// read and PV reads it as the TMEM A operand (tcgen05 TS form).  tcgen05 MMAs execute in
// issue order, so S_A(j+1) may be issued right behind PV_A(j) that reads the same columns,
// and s_full(j) fires only after every earlier MMA (including PV(j-1)) retired, which is
// what lets the softmax rescale O in place.
// Per score: one FFMA (scale folded into the exponent), one ex2.approx, one FADD, half a
// pack; O is rescaled only when the running max grows by more than 2^8 (exact).
// LSE is stored in the log2 domain with the softmax scale folded in (the backward's
// convention).
#include "common.cuh"
#include "sm100_ptx.cuh"
#include "tma_host.hpp"

namespace amdp {
namespace {

constexpr int FA_BQ = 256, FA_BKV = 128, FA_THREADS = 384;
#ifndef FA_POLY_PAIRS
#define FA_POLY_PAIRS 1  // of every 4 exponent pairs, this many are evaluated on the FMA pipe (1 measured best)
#endif
constexpr uint32_t TILE = 16384;  // one [128 rows][64 bf16] SW128 tile

// Diagnostics: when set (amdp_debug_attention_trace), CTA 0 records clock64() at each
// pipeline hand-off into this buffer (slot layout in scripts/attn_trace.py).
__device__ long long* g_fa_dbg = nullptr;
// Per-CTA (start ns, end ns, smid) when set (amdp_debug_attention_cta_times).
__device__ long long* g_fa_cta = nullptr;
#define FA_T(slot, j)                                                                        \
  do {                                                                                       \
    if (dbg_ != nullptr && (j) < 64) dbg_[(slot)*64 + (j)] = clock64(); \
  } while (0)

// head_dim 80 (GPT-2.7B) runs on the 128-wide layout: every row tile is two 64-column SW128
// boxes (the second box's columns 80-127 belong to the next head and are never used), the
// S = Q K^T reduction issues D/16 = 5 K-steps, and the PV / dV / dK / dQ MMAs use N = D = 80
// (an MN-major B operand of 64 + 16 columns across the two boxes).
template <int D>
struct FaSmem {
  static constexpr int NB = (D + 63) / 64;          // 64-wide column blocks per row tile
  static constexpr int KVS = NB == 2 ? 2 : 4;       // K / V ring depth
  static constexpr uint32_t Q = 0;                  // Q_A | Q_B
  static constexpr uint32_t K = Q + 2 * NB * TILE;
  static constexpr uint32_t V = K + KVS * NB * TILE;
  static constexpr uint32_t BAR = V + KVS * NB * TILE;
  static constexpr uint32_t BYTES = BAR + 256;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}


// P = 2^(S*scale - m) for one 128-column row held in registers, written as bf16 pairs over
// the first 64 TMEM columns of the S tile; returns the row sum.  Packed f32x2 arithmetic and
// one exponent pair in four on the FMA pipe keep issue slots and MUFU below the tensor time.
// MODE 0: every key; 1: causal diagonal block (key > qrow masked); 2: key padding (key >= qrow,
// here the sequence's valid key count, masked).
template <int MODE>
__device__ __forceinline__ float softmax_p_row(const uint32_t (&v)[FA_BKV], float scale_log2, float nm, int kbase,
                                               int qrow, uint32_t ts) {
  const float2 sc = make_float2(scale_log2, scale_log2), sh = make_float2(nm, nm);
  float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < FA_BKV / 32; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
      const float2 sv = make_float2(__uint_as_float(v[c * 32 + e]), __uint_as_float(v[c * 32 + e + 1]));
      const float2 x = __ffma2_rn(sv, sc, sh);
      float2 p;
      if (((e >> 1) & 3) < FA_POLY_PAIRS) {
        p = ex2_fma2(x);
      } else {
        p.x = ex2(x.x);
        p.y = ex2(x.y);
      }
      if (MODE == 1) {
        const int k0 = kbase + c * 32 + e;
        if (k0 > qrow) p.x = 0.f;
        if (k0 + 1 > qrow) p.y = 0.f;
      } else if (MODE == 2) {
        const int k0 = kbase + c * 32 + e;
        if (k0 >= qrow) p.x = 0.f;
        if (k0 + 1 >= qrow) p.y = 0.f;
      }
      if ((e >> 1) & 1) acc1 = __fadd2_rn(acc1, p);
      else acc0 = __fadd2_rn(acc0, p);
      __nv_bfloat162 t2 = __floats2bfloat162_rn(p.x, p.y);
      pk[e >> 1] = *reinterpret_cast<uint32_t*>(&t2);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            ts + c * 16),
        "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7]), "r"(pk[8]),
        "r"(pk[9]), "r"(pk[10]), "r"(pk[11]), "r"(pk[12]), "r"(pk[13]), "r"(pk[14]), "r"(pk[15])
        : "memory");
  }
  return (acc0.x + acc0.y) + (acc1.x + acc1.y);
}

// Persistent: one CTA per SM walks pair tiles in a snake order over the heavy-first tile list
// (causal tiles late in the sequence carry more KV blocks), so the per-CTA prologue (barrier
// init, TMEM alloc, first loads) is paid once and the next tile's Q/K loads and first S MMA
// overlap the previous tile's epilogue.
struct FaTile {
  int qp, h, b, nkv, last_a;
};
__device__ __forceinline__ int fa_tile_index(int it) {
  const int G = gridDim.x, c = blockIdx.x;
  return it * G + ((it & 1) ? (G - 1 - c) : c);
}
__device__ __forceinline__ FaTile fa_tile(int idx, int BH, int H, int n_qt, int seq, int causal) {
  FaTile t;
  t.qp = n_qt - 1 - idx / BH;  // heavy first
  const int hb = idx % BH;
  t.h = hb % H;
  t.b = hb / H;
  t.nkv = causal ? 2 * t.qp + 2 : seq / FA_BKV;  // blocks warpgroup B needs
  t.last_a = causal ? 2 * t.qp : t.nkv - 1;       // last block warpgroup A needs
  return t;
}

template <int D>
__global__ void __launch_bounds__(FA_THREADS, 1)
    fa_fwd_tc_kernel(const __grid_constant__ CUtensorMap qkv_map, bf16* __restrict__ out,
                     float* __restrict__ lse, int seq, int H, int BH, int n_qt, float scale_log2,
                     int causal, const int32_t* __restrict__ key_len) {
  using L = FaSmem<D>;
  constexpr int KVS = L::KVS;
  extern __shared__ uint8_t smem_raw[];
  long long* const dbg_ = blockIdx.x == 0 ? g_fa_dbg : nullptr;  // trace hook, read once
  long long* const cta_t = g_fa_cta;
  if (cta_t != nullptr && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    cta_t[3 * blockIdx.x] = static_cast<long long>(t);
    cta_t[3 * blockIdx.x + 2] = smid;
  }
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* q_empty = bar + 1;
  uint64_t* k_full = bar + 2;          // [KVS]
  uint64_t* k_empty = k_full + 4;      // [KVS]
  uint64_t* v_full = k_empty + 4;      // [KVS]
  uint64_t* v_empty = v_full + 4;      // [KVS]
  uint64_t* s_full = v_empty + 4;      // [2] per warpgroup
  uint64_t* p_full = s_full + 2;       // [2]
  uint64_t* pv_done = p_full + 2;      // [2]
  uint64_t* o_empty = pv_done + 2;     // [2] warpgroup has read O out of TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = n_qt * BH;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&qkv_map);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int s = 0; s < KVS; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&s_full[s], 1);
      ptx::mbar_init(&p_full[s], 128);
      ptx::mbar_init(&pv_done[s], 1);
      ptx::mbar_init(&o_empty[s], 128);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ptx::pdl_wait();
  ptx::pdl_trigger();
  if (dbg_ != nullptr && threadIdx.x == 0) dbg_[10 * 64] = clock64();
  // register split: the softmax warpgroups hold a whole 128-column S row in registers
  // (setmaxnreg placed inside each role branch so it dominates that role's code)
  if (warp == 0) {
    ptx::regs_dec<56>();
    if (lane == 0) {
      int kv = 0;  // KV blocks loaded by this CTA so far (ring position)
      for (int it = 0;; ++it) {
        const int idx = fa_tile_index(it);
        if (idx >= ntiles) break;
        const FaTile T = fa_tile(idx, BH, H, n_qt, seq, causal);
        const int row0 = T.b * seq;
        ptx::mbar_wait(q_empty, (it & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(q_full, 2 * L::NB * TILE);
        for (int t = 0; t < 2; ++t)
          for (int c = 0; c < L::NB; ++c)
            ptx::tma_load_2d(sm + L::Q + (t * L::NB + c) * TILE, &qkv_map, q_full, T.h * D + 64 * c,
                             row0 + T.qp * FA_BQ + 128 * t);
        // K_j runs ahead of V_j: S(j) needs K_j before PV(j) needs V_j
        for (int j = 0; j <= T.nkv; ++j) {
          if (j < T.nkv) {
            const int g = kv + j, st = g % KVS;
            ptx::mbar_wait(&k_empty[st], ((g / KVS) & 1) ^ 1);
            if (it == 0) FA_T(8, j);
            ptx::mbar_arrive_expect_tx(&k_full[st], L::NB * TILE);
            for (int c = 0; c < L::NB; ++c)
              ptx::tma_load_2d(sm + L::K + (st * L::NB + c) * TILE, &qkv_map, &k_full[st],
                               H * D + T.h * D + 64 * c, row0 + j * FA_BKV);
          }
          if (j > 0) {
            const int g = kv + j - 1, st = g % KVS;
            ptx::mbar_wait(&v_empty[st], ((g / KVS) & 1) ^ 1);
            if (it == 0) FA_T(9, j - 1);
            ptx::mbar_arrive_expect_tx(&v_full[st], L::NB * TILE);
            for (int c = 0; c < L::NB; ++c)
              ptx::tma_load_2d(sm + L::V + (st * L::NB + c) * TILE, &qkv_map, &v_full[st],
                               2 * H * D + T.h * D + 64 * c, row0 + (j - 1) * FA_BKV);
          }
        }
        kv += T.nkv;
      }
    }
  } else if (warp == 1) {
    ptx::regs_dec<56>();
    {  // warp-wide MMA issue (elect.sync inside the asm; see mma_bf16_*_w)
      constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, FA_BKV, false, false);
      constexpr uint32_t id_o = ptx::idesc_bf16_f32(128, D, false, true);
      const uint64_t dq0 = ptx::umma_desc_sw128(ptx::smem_u32(sm + L::Q), 16, 1024);
      const uint64_t dk0 = ptx::umma_desc_sw128(ptx::smem_u32(sm + L::K), 16, 1024);
      const uint64_t dv0 = ptx::umma_desc_sw128(ptx::smem_u32(sm + L::V), TILE, 1024);
      auto issue_s = [&](int w, int st) {  // S_w = Q_w K^T (K in ring stage st)
        const uint64_t dk = dk0 + ((st * L::NB * TILE) >> 4);
        const uint64_t dq = dq0 + ((w * L::NB * TILE) >> 4);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = ((kk >> 2) * TILE + (kk & 3) * 32) >> 4;
          ptx::mma_bf16_ss_w(tmem + w * 128, dq + off, dk + off, id_s, kk > 0 ? 1u : 0u);
        }
        ptx::mma_commit_w(&s_full[w]);
      };
      auto issue_pv = [&](int w, int st, bool first) {  // O_w += P_w V, P from TMEM
        ptx::tc_fence_after();
        const uint64_t dv = dv0 + ((st * L::NB * TILE) >> 4);
#pragma unroll
        for (int kk = 0; kk < FA_BKV / 16; ++kk)
          ptx::mma_bf16_ts_w(tmem + 256 + w * 128, tmem + w * 128 + kk * 8, dv + ((kk * 2048) >> 4), id_o,
                             (!first || kk > 0) ? 1u : 0u);
        ptx::mma_commit_w(&pv_done[w]);
      };
      int kv = 0, na = 0, nb = 0;  // KV blocks / A blocks / B blocks issued so far
      for (int it = 0;; ++it) {
        const int idx = fa_tile_index(it);
        if (idx >= ntiles) break;
        const FaTile T = fa_tile(idx, BH, H, n_qt, seq, causal);
        ptx::mbar_wait(q_full, it & 1);
        for (int j = 0; j <= T.nkv; ++j) {
          if (j < T.nkv) {
            const int g = kv + j;
            ptx::mbar_wait(&k_full[g % KVS], (g / KVS) & 1);
            if (it == 0) FA_T(0, j);
            ptx::tc_fence_after();
            if (j <= T.last_a) issue_s(0, g % KVS);
          }
          if (j > 0) {  // PV_B(j-1)
            const int g = kv + j - 1;
            ptx::mbar_wait(&v_full[g % KVS], (g / KVS) & 1);
            if (j == 1) ptx::mbar_wait(&o_empty[1], (it & 1) ^ 1);  // O_B of the previous tile read out
            ptx::mbar_wait(&p_full[1], (nb + j - 1) & 1);
            if (it == 0) FA_T(4, j - 1);
            issue_pv(1, g % KVS, j == 1);
            ptx::mma_commit_w(&v_empty[g % KVS]);  // PV_A(j-1) was issued before PV_B(j-1)
          }
          if (j < T.nkv) {
            const int g = kv + j;
            // start B's first softmax only once A's is done: the two warpgroups then keep
            // alternating between the MUFU and the tensor core instead of sharing both
            if (j == 0) ptx::mbar_wait(&p_full[0], na & 1);
            issue_s(1, g % KVS);
            ptx::mma_commit_w(&k_empty[g % KVS]);
            if (j == T.nkv - 1) ptx::mma_commit_w(q_empty);  // last read of this tile's Q
            if (j <= T.last_a) {
              ptx::mbar_wait(&v_full[g % KVS], (g / KVS) & 1);
              if (j == 0) ptx::mbar_wait(&o_empty[0], (it & 1) ^ 1);
              ptx::mbar_wait(&p_full[0], (na + j) & 1);
              if (it == 0) FA_T(3, j);
              issue_pv(0, g % KVS, j == 0);
            }
          }
        }
        kv += T.nkv;
        na += T.last_a + 1;
        nb += T.nkv;
      }
    }
  } else if (warp >= 4) {
    ptx::regs_inc<224>();
    const int wg = (warp - 4) >> 2;  // 0: rows 0-127 (A), 1: rows 128-255 (B)
    const int q = warp & 3;          // TMEM lane quadrant
    const int r = q * 32 + lane;
    const uint32_t lanes = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t ts = lanes + wg * 128;
    const uint32_t to = lanes + 256 + wg * 128;
    int nbase = 0;  // blocks this warpgroup processed in earlier tiles (barrier phases)
    for (int it = 0;; ++it) {
      const int idx = fa_tile_index(it);
      if (idx >= ntiles) break;
      const FaTile T = fa_tile(idx, BH, H, n_qt, seq, causal);
      const int qrow = T.qp * FA_BQ + 128 * wg + r;
      const int nblk = wg == 0 ? T.last_a + 1 : T.nkv;
      const int klen = key_len ? key_len[T.b] : seq;  // key padding (bidirectional models)
      float m_ref = -INFINITY, l = 0.f;
      for (int j = 0; j < nblk; ++j) {
        const bool diag = causal && j == nblk - 1;
        const bool lim = (j + 1) * FA_BKV > klen;  // keys >= klen in this block are padding
        ptx::mbar_wait(&s_full[wg], (nbase + j) & 1);  // also implies PV_wg(j-1) retired: O settled
        if (it == 0 && lane == 0 && q == 0) FA_T(5 + wg, j);
        ptx::tc_fence_after();
        // one pass over S: all 128 columns of this thread's row into registers
        uint32_t v[FA_BKV];
#pragma unroll
        for (int c = 0; c < FA_BKV / 32; ++c)
          ptx::tmem_ld_32x32b_x32(ts + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&v[c * 32]));
        ptx::tmem_ld_wait();
        float mx;
        {  // 8 independent max chains (a single chain is 64 dependent FMNMX deep)
          float m8[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) m8[t] = -INFINITY;
          if (diag) {
#pragma unroll
            for (int e = 0; e < FA_BKV; ++e)
              if (j * FA_BKV + e <= qrow) m8[e & 7] = fmaxf(m8[e & 7], __uint_as_float(v[e]));
          } else if (lim) {
#pragma unroll
            for (int e = 0; e < FA_BKV; ++e)
              if (j * FA_BKV + e < klen) m8[e & 7] = fmaxf(m8[e & 7], __uint_as_float(v[e]));
          } else {
#pragma unroll
            for (int e = 0; e < FA_BKV; e += 16)
#pragma unroll
              for (int t = 0; t < 8; ++t)
                m8[t] = fmaxf(m8[t], fmaxf(__uint_as_float(v[e + t]), __uint_as_float(v[e + 8 + t])));
          }
          mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        }
        const float m_new = fmaxf(m_ref, mx * scale_log2);
        if (it == 0 && lane == 0 && q == 0 && wg == 0) FA_T(12, j);
        if (j == 0) {
          m_ref = m_new;
        } else if (__any_sync(0xffffffffu, m_new > m_ref + 8.f)) {  // warp-collective TMEM ops
          const float alpha = ex2(m_ref - m_new);
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            ptx::tmem_ld_32x32b_x32(to + c * 32, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            ptx::tmem_st_32x32b_x32(to + c * 32, o);
          }
          if constexpr (D % 32 == 16) {
            uint32_t o[16];
            ptx::tmem_ld_32x32b_x16(to + (D / 32) * 32, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            ptx::tmem_st_32x32b_x16(to + (D / 32) * 32, o);
          }
          l *= alpha;
          m_ref = m_new;
        }
        const float nm = -m_ref;
        if (diag) l += softmax_p_row<1>(v, scale_log2, nm, j * FA_BKV, qrow, ts);
        else if (lim) l += softmax_p_row<2>(v, scale_log2, nm, j * FA_BKV, klen, ts);
        else l += softmax_p_row<0>(v, scale_log2, nm, j * FA_BKV, qrow, ts);
        if (it == 0 && lane == 0 && q == 0 && wg == 0) FA_T(13, j);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&p_full[wg]);
        if (it == 0 && lane == 0 && q == 0) FA_T(1 + wg, j);
      }
      ptx::mbar_wait(&pv_done[wg], (nbase + nblk - 1) & 1);
      ptx::tc_fence_after();
      const float inv = 1.f / l;
      bf16* orow = out + (static_cast<size_t>(T.b) * seq + qrow) * (static_cast<size_t>(H) * D) + T.h * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        ptx::tmem_ld_32x32b_x32(to + c * 32, o);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(o[8 * u + e]) * inv;
          store8(orow + c * 32 + 8 * u, f);
        }
      }
      if constexpr (D % 32 == 16) {
        uint32_t o[16];
        ptx::tmem_ld_32x32b_x16(to + (D / 32) * 32, o);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(o[8 * u + e]) * inv;
          store8(orow + (D / 32) * 32 + 8 * u, f);
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&o_empty[wg]);
      lse[(static_cast<size_t>(T.b) * H + T.h) * seq + qrow] = m_ref + log2f(l);
      nbase += nblk;
    }
  } else {
    ptx::regs_dec<56>();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
  if (cta_t != nullptr && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    cta_t[3 * blockIdx.x + 1] = static_cast<long long>(t);
  }
}

template <int D>
int launch_fa_fwd(const bf16* qkv, bf16* out, float* lse, int B, int S, int H, int causal, const int32_t* key_len,
                  cudaStream_t st) {
  CUtensorMap map;
  if (!tma_map_bf16_2d(&map, qkv, static_cast<uint64_t>(3) * H * D, static_cast<uint64_t>(B) * S,
                       static_cast<uint64_t>(3) * H * D, 64, 128))
    return AMDP_ERR_TMA;
  const size_t smem = FaSmem<D>::BYTES + 1024;
  auto k = fa_fwd_tc_kernel<D>;
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) {
      attr.store(0);
      return e;
    }
  }
  const int n_qt = S / FA_BQ;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  const int grid = std::min(n_qt * H * B, num_sms());
  cudaError_t e = launch_pdl(k, dim3(grid), dim3(FA_THREADS), smem, st, map, out, lse, S, H, H * B, n_qt, scale_log2,
                             causal, key_len);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

// Used by amdp_attention_fwd when the tensor-core path applies (seq % 256 == 0).
int attention_fwd_tc(const bf16* qkv, bf16* out, float* lse, int B, int S, int H, int D, int causal,
                     const int32_t* key_len, cudaStream_t st) {
  if (S % FA_BQ != 0) return AMDP_ERR_UNSUPPORTED;
  if (D == 128) return launch_fa_fwd<128>(qkv, out, lse, B, S, H, causal, key_len, st);
  if (D == 64) return launch_fa_fwd<64>(qkv, out, lse, B, S, H, causal, key_len, st);
  if (D == 80) return launch_fa_fwd<80>(qkv, out, lse, B, S, H, causal, key_len, st);
  return AMDP_ERR_UNSUPPORTED;
}

}  // namespace amdp

// Diagnostics hook (see g_fa_dbg): device buffer of >= 16 * 64 int64, or NULL to disable.
extern "C" int amdp_debug_attention_trace(long long* device_buf) {
  return cudaMemcpyToSymbol(amdp::g_fa_dbg, &device_buf, sizeof(device_buf));
}
extern "C" int amdp_debug_attention_cta_times(long long* device_buf) {
  return cudaMemcpyToSymbol(amdp::g_fa_cta, &device_buf, sizeof(device_buf));
}
