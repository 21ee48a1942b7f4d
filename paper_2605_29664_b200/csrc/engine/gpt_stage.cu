// GPT stage forward/backward as kernel sequences (see gpt_stage.hpp).
#include <algorithm>
#include <cmath>

#include "gpt_stage.hpp"
#include "ktimer.hpp"

namespace amdp {

namespace {
constexpr int64_t kAlign = 64;  // elements; keeps every tensor 128-B aligned for TMA
int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct Carver {
  uint8_t* p;
  size_t used = 0;
  template <class T>
  T* take(size_t n) {
    T* r = reinterpret_cast<T*>(p ? p + used : nullptr);
    used += (n * sizeof(T) + 255) & ~static_cast<size_t>(255);
    return r;
  }
};

// One stage contraction; timed by class (forward / activation-gradient / weight-gradient)
// when the executor's kernel timer is on.
int gemm_t(KTimer* kt, int M, int N, int K, const void* A, int lda, bool amn, const void* B, int ldb,
           bool bmn, void* C, int ldc, int epi, cudaStream_t s, const void* aux = nullptr,
           int ld_aux = 0, void* C2 = nullptr, int ldc2 = 0, int cls = -1, float* rowdot = nullptr,
           int rowdot_seg = 0, int rowdot_seq = 0) {
  amdp_gemm_args a{M, N, K, A, lda, amn ? 1 : 0, B, ldb, bmn ? 1 : 0, C, ldc, aux, ld_aux, C2, ldc2,
                   epi, 1.0f, rowdot, rowdot_seg, rowdot_seq};
  if (cls < 0) cls = epi == AMDP_EPI_ACCUM_F32 ? K_GEMM_WGRAD : (bmn ? K_GEMM_DGRAD : K_GEMM_FWD);
  if (kt) kt->begin(cls, 2.0 * M * N * static_cast<double>(K), 0, s);
  const int rc = amdp_gemm(&a, reinterpret_cast<amdp_stream_t>(s));
  if (kt) kt->end(s);
  return rc;
}
// dst[c][r] = src[r][c] for a [rows][cols] bf16 matrix (rows, cols multiples of 8): 64x64
// tiles through shared memory, 16-byte global loads and stores (8 bf16 per thread per access).
__global__ void __launch_bounds__(256) transpose_bf16_kernel(const uint16_t* __restrict__ src,
                                                             uint16_t* __restrict__ dst, int rows, int cols) {
  __shared__ uint16_t tile[64][72];  // +8 columns: 16-byte aligned rows, fewer bank conflicts
  const int c0 = blockIdx.x * 64, r0 = blockIdx.y * 64;
  const int t = threadIdx.x;
  for (int i = t; i < 64 * 8; i += 256) {  // 64 rows x 8 chunks of 8 columns
    const int r = i >> 3, c = (i & 7) * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r0 + r < rows && c0 + c < cols) v = *reinterpret_cast<const uint4*>(src + static_cast<size_t>(r0 + r) * cols + c0 + c);
    *reinterpret_cast<uint4*>(&tile[r][c]) = v;
  }
  __syncthreads();
  for (int i = t; i < 64 * 8; i += 256) {  // 64 output rows (source columns) x 8 chunks of 8 rows
    const int c = i >> 3, r = (i & 7) * 8;
    if (c0 + c >= cols || r0 + r >= rows) continue;
    uint4 o;
    o.x = tile[r][c] | (static_cast<uint32_t>(tile[r + 1][c]) << 16);
    o.y = tile[r + 2][c] | (static_cast<uint32_t>(tile[r + 3][c]) << 16);
    o.z = tile[r + 4][c] | (static_cast<uint32_t>(tile[r + 5][c]) << 16);
    o.w = tile[r + 6][c] | (static_cast<uint32_t>(tile[r + 7][c]) << 16);
    *reinterpret_cast<uint4*>(dst + static_cast<size_t>(c0 + c) * rows + r0 + r) = o;
  }
}
}  // namespace

int GptStage::refresh_transposed(cudaStream_t s) const {
  if (!wt || d_.fp32) return 0;  // fp32 mode reads `master` with MN-major operands
  int launched = 0;
  auto tr = [&](const ParamRef& p) {
    dim3 grid((p.cols + 63) / 64, (p.rows + 63) / 64);
    transpose_bf16_kernel<<<grid, 256, 0, s>>>(w + p.off, wt + p.off, p.rows, p.cols);
    ++launched;
  };
  for (const LayerParams& P : layers_) {
    tr(P.qkv);
    tr(P.o);
    tr(P.fc1);
    tr(P.fc2);
  }
  if (last()) tr(head_);
  return cudaGetLastError() == cudaSuccess ? launched : -1;
}

GptStage::GptStage(const Dims& d, int stage, int depth, int l0, int l1)
    : d_(d), stage_(stage), depth_(depth), l0_(l0), l1_(l1) {
  const float std = 0.02f;
  const float proj_std = std / std::sqrt(2.0f * static_cast<float>(d.L));
  if (first()) {
    wte_ = add("wte", d.V, d.h, 0, 0, std);
    wpe_ = add("wpe", d.S, d.h, 1, 0, std);
  }
  for (int l = l0; l < l1; ++l) {
    const int g = 16 + 8 * l;
    const std::string p = "layer" + std::to_string(l) + ".";
    LayerParams lp;
    lp.ln1_g = add(p + "ln1.gamma", 1, d.h, g + 0, 1, 0.f);
    lp.ln1_b = add(p + "ln1.beta", 1, d.h, g + 1, 2, 0.f);
    lp.qkv = add(p + "attn.qkv", 3 * d.h, d.h, g + 2, 0, std);
    lp.o = add(p + "attn.out", d.h, d.h, g + 3, 0, proj_std);
    lp.ln2_g = add(p + "ln2.gamma", 1, d.h, g + 4, 1, 0.f);
    lp.ln2_b = add(p + "ln2.beta", 1, d.h, g + 5, 2, 0.f);
    lp.fc1 = add(p + "mlp.fc1", d.ffn, d.h, g + 6, 0, std);
    lp.fc2 = add(p + "mlp.fc2", d.h, d.ffn, g + 7, 0, proj_std);
    layers_.push_back(lp);
  }
  if (last()) {
    lnf_g_ = add("lnf.gamma", 1, d.h, 2, 1, 0.f);
    lnf_b_ = add("lnf.beta", 1, d.h, 3, 2, 0.f);
    head_ = add("head", d.V, d.h, 4, 0, std);
  }
}

ParamRef GptStage::add(const std::string& name, int rows, int cols, int gidx, int init, float std) {
  ParamRef r;
  r.name = name;
  r.off = numel_;
  r.rows = rows;
  r.cols = cols;
  r.global_index = gidx;
  r.init = init;
  r.std = std;
  numel_ = round_up(numel_ + r.numel(), kAlign);
  all_.push_back(r);
  return r;
}

size_t GptStage::slot_bytes() const {
  Carver c{nullptr};
  SlotActs a;
  (void)a;
  const size_t T = static_cast<size_t>(d_.T), h = static_cast<size_t>(d_.h);
  const size_t E = d_.act_bytes() / 2;  // uint16 units per activation element
  if (first()) c.take<uint16_t>(E * T * h);
  for (int l = l0_; l < l1_; ++l) {
    if (l > l0_) c.take<uint16_t>(E * T * h);  // x
    c.take<uint16_t>(E * T * h);               // ln1
    c.take<uint16_t>(E * T * 3 * h);           // qkv
    if (!d_.recompute) c.take<uint16_t>(E * T * h);  // o
    c.take<uint16_t>(E * T * h);               // hmid
    c.take<uint16_t>(E * T * h);               // ln2
    c.take<uint16_t>(E * T * d_.ffn);          // u
    if (!d_.recompute) c.take<uint16_t>(E * T * d_.ffn);  // f
    c.take<float>(T);
    c.take<float>(T);
    c.take<float>(T);
    c.take<float>(T);
    c.take<float>(static_cast<size_t>(d_.B) * d_.heads * d_.S);  // lse
  }
  if (last()) {
    c.take<uint16_t>(E * T * h);
    c.take<uint16_t>(E * T * h);
    c.take<float>(T);
    c.take<float>(T);
    c.take<uint16_t>(E * T * static_cast<size_t>(d_.V));
  }
  return c.used;
}

SlotActs GptStage::carve_slot(uint8_t* base) const {
  Carver c{base};
  SlotActs a;
  const size_t T = static_cast<size_t>(d_.T), h = static_cast<size_t>(d_.h);
  const size_t E = d_.act_bytes() / 2;  // uint16 units per activation element
  if (first()) a.x0 = c.take<uint16_t>(E * T * h);
  for (int l = l0_; l < l1_; ++l) {
    LayerActs la;
    if (l > l0_) la.x = c.take<uint16_t>(E * T * h);
    la.ln1 = c.take<uint16_t>(E * T * h);
    la.qkv = c.take<uint16_t>(E * T * 3 * h);
    la.o = d_.recompute ? nullptr : c.take<uint16_t>(E * T * h);
    la.hmid = c.take<uint16_t>(E * T * h);
    la.ln2 = c.take<uint16_t>(E * T * h);
    la.u = c.take<uint16_t>(E * T * d_.ffn);
    la.f = d_.recompute ? nullptr : c.take<uint16_t>(E * T * d_.ffn);
    la.ln1_mean = c.take<float>(T);
    la.ln1_rstd = c.take<float>(T);
    la.ln2_mean = c.take<float>(T);
    la.ln2_rstd = c.take<float>(T);
    la.lse = c.take<float>(static_cast<size_t>(d_.B) * d_.heads * d_.S);
    a.layers.push_back(la);
  }
  if (last()) {
    a.xf = c.take<uint16_t>(E * T * h);
    a.lnf = c.take<uint16_t>(E * T * h);
    a.lnf_mean = c.take<float>(T);
    a.lnf_rstd = c.take<float>(T);
    a.logits = c.take<uint16_t>(E * T * static_cast<size_t>(d_.V));
  }
  return a;
}

namespace {
struct Ws {
  uint16_t *g0, *g1, *dU, *dqkv, *dtmp, *dhmid;
  float* attn;
  uint8_t* ln;
  uint16_t *rc_o = nullptr, *rc_f = nullptr;  // recompute: this layer's o and f
  float* rows = nullptr;  // per-token scratch: CE row losses / sorted embedding keys
};
Ws carve_ws(const Dims& d, uint8_t* base) {
  Carver c{base};
  const size_t T = static_cast<size_t>(d.T), h = static_cast<size_t>(d.h);
  const size_t E = d.act_bytes() / 2;  // uint16 units per activation element
  Ws w;
  w.g0 = c.take<uint16_t>(E * T * h);
  w.g1 = c.take<uint16_t>(E * T * h);
  w.dU = c.take<uint16_t>(E * T * d.ffn);
  w.dqkv = c.take<uint16_t>(E * T * 3 * h);
  w.dtmp = c.take<uint16_t>(E * T * h);
  w.dhmid = c.take<uint16_t>(E * T * h);
  w.attn = c.take<float>(std::max(amdp_attention_bwd_workspace_causal(d.B, d.S, d.heads, d.hd, d.causal ? 1 : 0),
                                 amdp_f32_attention_bwd_workspace(d.B, d.S, d.heads)) / sizeof(float) + 1);
  w.ln = c.take<uint8_t>(amdp_layernorm_bwd_workspace(d.T, d.h));
  w.rows = c.take<float>(T);
  if (d.recompute) {
    w.rc_o = c.take<uint16_t>(E * T * h);
    w.rc_f = c.take<uint16_t>(E * T * d.ffn);
  }
  return w;
}
}  // namespace

size_t GptStage::workspace_bytes(const Dims& d) {
  Carver c{nullptr};
  const size_t T = static_cast<size_t>(d.T), h = static_cast<size_t>(d.h);
  const size_t E = d.act_bytes() / 2;  // uint16 units per activation element
  c.take<uint16_t>(E * T * h);
  c.take<uint16_t>(E * T * h);
  c.take<uint16_t>(E * T * d.ffn);
  c.take<uint16_t>(E * T * 3 * h);
  c.take<uint16_t>(E * T * h);
  c.take<uint16_t>(E * T * h);
  c.take<float>(std::max(amdp_attention_bwd_workspace_causal(d.B, d.S, d.heads, d.hd, d.causal ? 1 : 0),
                                 amdp_f32_attention_bwd_workspace(d.B, d.S, d.heads)) / sizeof(float) + 1);
  c.take<uint8_t>(amdp_layernorm_bwd_workspace(d.T, d.h));
  c.take<float>(T);
  if (d.recompute) {
    c.take<uint16_t>(E * T * h);
    c.take<uint16_t>(E * T * d.ffn);
  }
  return c.used;
}

#define AMDP_TRY(cls, fl, by, expr, nk)   \
  do {                                    \
    if (kt) kt->begin((cls), (fl), (by), s); \
    const int _r = (expr);                \
    if (kt) kt->end(s);                   \
    if (_r != 0) {                        \
      *rc = _r;                           \
      return launched;                    \
    }                                     \
    launched += (nk);                     \
  } while (0)

#define AMDP_GEMM(call, nk)   \
  do {                        \
    const int _r = (call);    \
    if (_r != 0) {            \
      *rc = _r;               \
      return launched;        \
    }                         \
    launched += (nk);         \
  } while (0)

int GptStage::flush_ln_grads(cudaStream_t s, int* rc) const {
  int launched = 0;
  *rc = 0;
  if (!ln_part) return 0;
  const int parts = ln_parts(), h = d_.h;
  for (int k = 0; k < ln_count(); ++k) {
    const bool fin = last() && k == ln_count() - 1;
    const LayerParams* P = fin ? nullptr : &layers_[static_cast<size_t>(k / 2)];
    const ParamRef& g = fin ? lnf_g_ : (k % 2 ? P->ln2_g : P->ln1_g);
    const ParamRef& b = fin ? lnf_b_ : (k % 2 ? P->ln2_b : P->ln1_b);
    AMDP_TRY(K_LAYERNORM, 0, 8.0 * parts * h, amdp_layernorm_dgb_flush(ln_part + static_cast<size_t>(k) * parts * 2 * h, parts,
                                                                        h, grad + g.off, grad + b.off,
                                                                        reinterpret_cast<amdp_stream_t>(s)), 1);
  }
  return launched;
}

std::vector<std::pair<int64_t, int64_t>> GptStage::segments() const {
  std::vector<int64_t> starts;
  if (first()) starts.push_back(0);
  for (const LayerParams& P : layers_) starts.push_back(P.ln1_g.off);
  if (last()) starts.push_back(lnf_g_.off);
  std::vector<std::pair<int64_t, int64_t>> out;
  for (size_t k = 0; k < starts.size(); ++k)
    out.emplace_back(starts[k], (k + 1 < starts.size() ? starts[k + 1] : numel_) - starts[k]);
  return out;
}

int GptStage::forward(const SlotActs& a, const int32_t* tokens, const int32_t* labels,
                      const uint16_t* in, uint16_t* out, float* loss_sum, float loss_scale, uint8_t* wsb,
                      cudaStream_t s, int* rc, const cudaEvent_t* seg_ready, const int32_t* key_len) const {
  if (d_.fp32)
    return forward_f32(a, tokens, labels, reinterpret_cast<const float*>(in), reinterpret_cast<float*>(out), loss_sum,
                       loss_scale, wsb, s, rc, seg_ready, key_len);
  int seg = 0;  // next segment to wait for
  auto wait_seg = [&]() {
    if (seg_ready) cudaStreamWaitEvent(s, seg_ready[seg], 0);
    ++seg;
  };
  const Ws ws = carve_ws(d_, wsb);
  int launched = 0;
  *rc = 0;
  auto st = reinterpret_cast<amdp_stream_t>(s);
  const int T = d_.T, h = d_.h;
  const uint16_t* x = in;
  if (first()) {
    wait_seg();
    AMDP_TRY(K_EMBED, 0, 6.0 * T * h, amdp_embedding_fwd(tokens, w + wte_.off, w + wpe_.off, a.x0, T, d_.S, h, st), 1);
    x = a.x0;
  }
  for (int li = 0; li < l1_ - l0_; ++li) {
    const LayerParams& P = layers_[static_cast<size_t>(li)];
    LayerActs A = a.layers[static_cast<size_t>(li)];
    if (d_.recompute) {  // o and f live in the workspace, rebuilt by the backward
      A.o = ws.rc_o;
      A.f = ws.rc_f;
    }
    wait_seg();
    AMDP_TRY(K_LAYERNORM, 0, 4.0 * T * h, amdp_layernorm_fwd(x, master + P.ln1_g.off, master + P.ln1_b.off, A.ln1, A.ln1_mean,
                                A.ln1_rstd, T, h, d_.ln_eps, st), 1);
    AMDP_GEMM(gemm_t(kt, T, 3 * h, h, A.ln1, h, false, w + P.qkv.off, h, false, A.qkv, 3 * h,
                  AMDP_EPI_STORE_BF16, s), 1);
    AMDP_TRY(K_ATTN_FWD, attn_fwd_flops(), 0, amdp_attention_fwd(A.qkv, A.o, A.lse, d_.B, d_.S, d_.heads, d_.hd, d_.causal ? 1 : 0, key_len, st), 1);
    AMDP_GEMM(gemm_t(kt, T, h, h, A.o, h, false, w + P.o.off, h, false, A.hmid, h, AMDP_EPI_RESIDUAL, s, x, h), 1);
    AMDP_TRY(K_LAYERNORM, 0, 4.0 * T * h, amdp_layernorm_fwd(A.hmid, master + P.ln2_g.off, master + P.ln2_b.off, A.ln2, A.ln2_mean,
                                A.ln2_rstd, T, h, d_.ln_eps, st), 1);
    AMDP_GEMM(gemm_t(kt, T, d_.ffn, h, A.ln2, h, false, w + P.fc1.off, h, false, A.f, d_.ffn, AMDP_EPI_GELU, s,
                  nullptr, 0, A.u, d_.ffn), 1);
    uint16_t* nx;
    if (li + 1 < l1_ - l0_) nx = a.layers[static_cast<size_t>(li) + 1].x;
    else nx = last() ? a.xf : out;
    AMDP_GEMM(gemm_t(kt, T, h, d_.ffn, A.f, d_.ffn, false, w + P.fc2.off, d_.ffn, false, nx, h, AMDP_EPI_RESIDUAL,
                  s, A.hmid, h), 1);
    x = nx;
  }
  if (last()) {
    wait_seg();
    AMDP_TRY(K_LAYERNORM, 0, 4.0 * T * h, amdp_layernorm_fwd(a.xf, master + lnf_g_.off, master + lnf_b_.off, a.lnf, a.lnf_mean,
                                a.lnf_rstd, T, h, d_.ln_eps, st), 1);
    AMDP_GEMM(gemm_t(kt, T, d_.V, h, a.lnf, h, false, w + head_.off, h, false, a.logits, d_.V,
                  AMDP_EPI_STORE_BF16, s), 1);
    AMDP_TRY(K_XENT, 0, 6.0 * T * d_.V, amdp_xent_fwd_bwd(a.logits, labels, loss_sum, ws.rows, T, d_.V, d_.V, loss_scale, st), 1);
  }
  return launched;
}

// Weight-gradient GEMMs run on `side` so they fill the wave-quantisation tails of the
// activation-gradient chain on `s` (most stage GEMMs have N = h = 2048: 3.5 waves of
// 256x256 pair tiles on 148 SMs).  Events order every hand-off; the task ends with `s`
// joined to `side`, so slot activations and gradient buffers are quiescent afterwards.
int GptStage::backward(const SlotActs& a, const int32_t* tokens, const uint16_t* in, const uint16_t* gin,
                       uint16_t* gout, uint8_t* wsb, cudaStream_t s, const SideStream& ss, int* rc,
                       const int32_t* key_len) const {
  if (d_.fp32)
    return backward_f32(a, tokens, reinterpret_cast<const float*>(in), reinterpret_cast<const float*>(gin),
                        reinterpret_cast<float*>(gout), wsb, s, rc, key_len);
  int launched = 0;
  *rc = 0;
  auto st = reinterpret_cast<amdp_stream_t>(s);
  const int T = d_.T, h = d_.h, F = d_.ffn;
  const Ws ws = carve_ws(d_, wsb);
  cudaStream_t sd = ss.side ? ss.side : s;
  // LayerNorm k's backward (k = 2 li / 2 li + 1 for a layer's ln1 / ln2, the last one for the
  // final LayerNorm): deferred parameter gradients when ln_part is set
  auto ln_bwd = [&](int k, const uint16_t* dy, const uint16_t* xin, const ParamRef& pg, const ParamRef& pb,
                    const float* mean, const float* rstd, const uint16_t* resid, uint16_t* dx, void* lnws,
                    amdp_stream_t stream) {
    if (ln_part)
      return amdp_layernorm_bwd_rows(dy, xin, master + pg.off, mean, rstd, resid, dx,
                                     ln_part + static_cast<size_t>(k) * ln_parts() * 2 * h, T, h, stream);
    return amdp_layernorm_bwd(dy, xin, master + pg.off, mean, rstd, resid, dx, grad + pg.off, grad + pb.off, lnws, T,
                              h, stream);
  };
  static const bool no_fuse = getenv("AMDP_NO_DELTA_FUSION") != nullptr;
  const bool fuse_delta = !no_fuse && d_.hd % 64 == 0 && amdp_attention_bwd_delta_supported(d_.S, d_.hd);
  auto hand = [&](cudaEvent_t e, cudaStream_t from, cudaStream_t to) {
    if (from == to) return;
    cudaEventRecord(e, from);
    cudaStreamWaitEvent(to, e, 0);
  };
  enum { E_G, E_DU, E_DH, E_DQ, F_G, F_DU, F_DH, F_DQ, E_HEAD, F_END };
  const uint16_t* g = gin;
  if (last()) {
    // a.logits already holds dloss/dlogits (scale 1/T), written by the forward's CE pass
    hand(ss.ev[E_HEAD], s, sd);
    AMDP_GEMM(gemm_t(kt, d_.V, h, T, a.logits, d_.V, true, a.lnf, h, true, grad + head_.off, h,
                     AMDP_EPI_ACCUM_F32, sd), 1);
    AMDP_GEMM(gemm_t(kt, T, h, d_.V, a.logits, d_.V, false, wt + head_.off, d_.V, false, ws.dtmp, h,
                     AMDP_EPI_STORE_BF16, s, nullptr, 0, nullptr, 0, K_GEMM_DGRAD), 1);
    AMDP_TRY(K_LAYERNORM, 0, 8.0 * T * h, ln_bwd(ln_count() - 1, ws.dtmp, a.xf, lnf_g_, lnf_b_, a.lnf_mean, a.lnf_rstd,
                                                 nullptr, ws.g0, ws.ln, st), ln_part ? 1 : 2);
    g = ws.g0;
  }
  for (int li = l1_ - l0_ - 1; li >= 0; --li) {
    const LayerParams& P = layers_[static_cast<size_t>(li)];
    LayerActs A = a.layers[static_cast<size_t>(li)];
    if (d_.recompute) {  // o and f live in the workspace, rebuilt by the backward
      A.o = ws.rc_o;
      A.f = ws.rc_f;
    }
    const uint16_t* x = li > 0 ? A.x : (first() ? a.x0 : in);
    // y = hmid + f W2^T
    if (d_.recompute) {  // f = gelu(u): weight-independent, exact under staleness
      // the layer above's fc2 weight gradient (side stream) has finished reading the shared f
      if (sd != s) cudaStreamWaitEvent(s, ss.ev[F_G], 0);
      AMDP_TRY(K_GELU, 0, 4.0 * T * F, amdp_gelu_fwd(A.u, A.f, static_cast<int64_t>(T) * F, st), 1);
    }
    hand(ss.ev[E_G], s, sd);
    AMDP_GEMM(gemm_t(kt, h, F, T, g, h, true, A.f, F, true, grad + P.fc2.off, F, AMDP_EPI_ACCUM_F32, sd), 1);
    if (sd != s) cudaEventRecord(ss.ev[F_G], sd);
    if (sd != s) cudaStreamWaitEvent(s, ss.ev[F_DU], 0);  // previous layer's dW1 done with dU
    AMDP_GEMM(gemm_t(kt, T, F, h, g, h, false, wt + P.fc2.off, h, false, ws.dU, F, AMDP_EPI_GELU_BWD, s, A.u, F,
                     nullptr, 0, K_GEMM_DGRAD), 1);
    hand(ss.ev[E_DU], s, sd);
    // f = gelu(ln2 W1^T)
    AMDP_GEMM(gemm_t(kt, F, h, T, ws.dU, F, true, A.ln2, h, true, grad + P.fc1.off, h, AMDP_EPI_ACCUM_F32, sd), 1);
    if (sd != s) cudaEventRecord(ss.ev[F_DU], sd);
    AMDP_GEMM(gemm_t(kt, T, h, F, ws.dU, F, false, wt + P.fc1.off, F, false, ws.dtmp, h, AMDP_EPI_STORE_BF16, s,
                     nullptr, 0, nullptr, 0, K_GEMM_DGRAD), 1);
    // ln2 = LN(hmid); dhmid = g + LN'(dln2)
    if (sd != s) cudaStreamWaitEvent(s, ss.ev[F_DH], 0);  // previous layer's dWo done with dhmid
    AMDP_TRY(K_LAYERNORM, 0, 8.0 * T * h, ln_bwd(2 * li + 1, ws.dtmp, A.hmid, P.ln2_g, P.ln2_b, A.ln2_mean, A.ln2_rstd, g,
                                                 ws.dhmid, ws.ln, st), ln_part ? 1 : 2);
    // o = attention(qkv) when recomputing: deterministic (rewrites the same lse), issued before
    // the hand-off so the side stream's out-proj weight gradient reads the rebuilt o; its
    // previous reader (the layer above's) finished before F_DH, waited for above
    if (d_.recompute)
      AMDP_TRY(K_ATTN_FWD, attn_fwd_flops(), 0, amdp_attention_fwd(A.qkv, A.o, A.lse, d_.B, d_.S, d_.heads, d_.hd,
                                                                   d_.causal ? 1 : 0, key_len, st), 1);
    hand(ss.ev[E_DH], s, sd);
    // hmid = x + o Wo^T
    AMDP_GEMM(gemm_t(kt, h, h, T, ws.dhmid, h, true, A.o, h, true, grad + P.o.off, h, AMDP_EPI_ACCUM_F32, sd), 1);
    if (sd != s) cudaEventRecord(ss.ev[F_DH], sd);
    // dO = dhmid Wo; its epilogue also forms the attention backward's delta = rowsum(dO * O)
    // per head (AMDP_EPI_ROWDOT) instead of a separate pass over dO and O
    if (fuse_delta) {
      AMDP_GEMM(gemm_t(kt, T, h, h, ws.dhmid, h, false, wt + P.o.off, h, false, ws.dtmp, h, AMDP_EPI_ROWDOT, s,
                       A.o, h, nullptr, 0, K_GEMM_DGRAD, ws.attn, d_.hd, d_.S), 1);
    } else {
      AMDP_GEMM(gemm_t(kt, T, h, h, ws.dhmid, h, false, wt + P.o.off, h, false, ws.dtmp, h, AMDP_EPI_STORE_BF16, s,
                       nullptr, 0, nullptr, 0, K_GEMM_DGRAD), 1);
    }
    if (sd != s) cudaStreamWaitEvent(s, ss.ev[F_DQ], 0);  // previous layer's dWqkv done with dqkv
    if (fuse_delta) {
      // workspace layout of amdp_attention_bwd_workspace_causal: delta, then the dS^T scratch
      uint8_t* scratch = reinterpret_cast<uint8_t*>(ws.attn) +
                         ((static_cast<size_t>(d_.B) * d_.S * d_.heads * sizeof(float) + 255) & ~static_cast<size_t>(255));
      AMDP_TRY(K_ATTN_BWD, 2.5 * attn_fwd_flops(), 0, amdp_attention_bwd_delta_ws(A.qkv, ws.dtmp, A.lse, ws.attn, ws.dqkv,
                                  scratch, d_.B, d_.S, d_.heads, d_.hd, d_.causal ? 1 : 0, key_len, st), 2);
    } else {
      AMDP_TRY(K_ATTN_BWD, 2.5 * attn_fwd_flops(), 0, amdp_attention_bwd(A.qkv, A.o, ws.dtmp, A.lse, ws.dqkv, ws.attn, d_.B, d_.S, d_.heads, d_.hd,
                                  d_.causal ? 1 : 0, key_len, st), 3);
    }
    hand(ss.ev[E_DQ], s, sd);
    // qkv = ln1 Wqkv^T
    AMDP_GEMM(gemm_t(kt, 3 * h, h, T, ws.dqkv, 3 * h, true, A.ln1, h, true, grad + P.qkv.off, h,
                     AMDP_EPI_ACCUM_F32, sd), 1);
    if (sd != s) cudaEventRecord(ss.ev[F_DQ], sd);
    AMDP_GEMM(gemm_t(kt, T, h, 3 * h, ws.dqkv, 3 * h, false, wt + P.qkv.off, 3 * h, false, ws.dtmp, h,
                     AMDP_EPI_STORE_BF16, s, nullptr, 0, nullptr, 0, K_GEMM_DGRAD), 1);
    uint16_t* gn = (li == 0 && !first()) ? gout : (g == ws.g0 ? ws.g1 : ws.g0);
    if (sd != s) cudaStreamWaitEvent(s, ss.ev[F_G], 0);  // dW2 of the layer that read gn's buffer
    AMDP_TRY(K_LAYERNORM, 0, 8.0 * T * h, ln_bwd(2 * li, ws.dtmp, x, P.ln1_g, P.ln1_b, A.ln1_mean, A.ln1_rstd, ws.dhmid, gn,
                                                 ws.ln, st), ln_part ? 1 : 2);
    g = gn;
  }
  if (first()) AMDP_TRY(K_EMBED, 0, 10.0 * T * h, amdp_embedding_bwd(tokens, g, grad + wte_.off, grad + wpe_.off, ws.rows, T, d_.S, h, st), 2);
  hand(ss.ev[F_END], sd, s);  // join: weight gradients complete before the task ends
  return launched;
}

// ------------------------------------------------------------------ fp32 validation mode
// The same stage math as forward() / backward() above on fp32 tensors (the slot and workspace
// pointers address floats), weights read from the fp32 master, every kernel an amdp_f32_*
// one, all on stream `s` in a fixed order (no side stream): bitwise reproducible.
namespace {
int gemm32(KTimer* kt, int M, int N, int K, const float* A, int lda, bool amn, const float* B, int ldb, bool bmn,
           float* C, int ldc, int epi, cudaStream_t s, const float* aux = nullptr, int ld_aux = 0,
           float* C2 = nullptr, int ldc2 = 0, int cls = -1) {
  amdp_gemm_args a{M, N, K, A, lda, amn ? 1 : 0, B, ldb, bmn ? 1 : 0, C, ldc, aux, ld_aux, C2, ldc2,
                   epi, 1.0f, nullptr, 0, 0};
  if (cls < 0) cls = epi == AMDP_EPI_ACCUM_F32 ? K_GEMM_WGRAD : (bmn ? K_GEMM_DGRAD : K_GEMM_FWD);
  if (kt) kt->begin(cls, 2.0 * M * N * static_cast<double>(K), 0, s);
  const int rc = amdp_f32_gemm(&a, reinterpret_cast<amdp_stream_t>(s));
  if (kt) kt->end(s);
  return rc;
}
inline float* F(uint16_t* p) { return reinterpret_cast<float*>(p); }
inline const float* F(const uint16_t* p) { return reinterpret_cast<const float*>(p); }
}  // namespace

int GptStage::forward_f32(const SlotActs& a, const int32_t* tokens, const int32_t* labels, const float* in,
                          float* out, float* loss_sum, float loss_scale, uint8_t* wsb, cudaStream_t s, int* rc,
                          const cudaEvent_t* seg_ready, const int32_t* key_len) const {
  int seg = 0;
  auto wait_seg = [&]() {
    if (seg_ready) cudaStreamWaitEvent(s, seg_ready[seg], 0);
    ++seg;
  };
  const Ws ws = carve_ws(d_, wsb);
  int launched = 0;
  *rc = 0;
  auto st = reinterpret_cast<amdp_stream_t>(s);
  const int T = d_.T, h = d_.h;
  const float* W = master;
  const float* x = in;
  if (first()) {
    wait_seg();
    AMDP_TRY(K_EMBED, 0, 12.0 * T * h, amdp_f32_embedding_fwd(tokens, W + wte_.off, W + wpe_.off, F(a.x0), T, d_.S, h, st), 1);
    x = F(a.x0);
  }
  for (int li = 0; li < l1_ - l0_; ++li) {
    const LayerParams& P = layers_[static_cast<size_t>(li)];
    const LayerActs& A = a.layers[static_cast<size_t>(li)];
    wait_seg();
    AMDP_TRY(K_LAYERNORM, 0, 8.0 * T * h, amdp_f32_layernorm_fwd(x, W + P.ln1_g.off, W + P.ln1_b.off, F(A.ln1), A.ln1_mean,
                                                                A.ln1_rstd, T, h, d_.ln_eps, st), 1);
    AMDP_GEMM(gemm32(kt, T, 3 * h, h, F(A.ln1), h, false, W + P.qkv.off, h, false, F(A.qkv), 3 * h, AMDP_EPI_STORE_F32, s), 1);
    AMDP_TRY(K_ATTN_FWD, attn_fwd_flops(), 0, amdp_f32_attention_fwd(F(A.qkv), F(A.o), A.lse, d_.B, d_.S, d_.heads, d_.hd,
                                                                     d_.causal ? 1 : 0, key_len, st), 1);
    AMDP_GEMM(gemm32(kt, T, h, h, F(A.o), h, false, W + P.o.off, h, false, F(A.hmid), h, AMDP_EPI_RESIDUAL, s, x, h), 1);
    AMDP_TRY(K_LAYERNORM, 0, 8.0 * T * h, amdp_f32_layernorm_fwd(F(A.hmid), W + P.ln2_g.off, W + P.ln2_b.off, F(A.ln2),
                                                                A.ln2_mean, A.ln2_rstd, T, h, d_.ln_eps, st), 1);
    AMDP_GEMM(gemm32(kt, T, d_.ffn, h, F(A.ln2), h, false, W + P.fc1.off, h, false, F(A.f), d_.ffn, AMDP_EPI_GELU, s,
                     nullptr, 0, F(A.u), d_.ffn), 1);
    float* nx;
    if (li + 1 < l1_ - l0_) nx = F(a.layers[static_cast<size_t>(li) + 1].x);
    else nx = last() ? F(a.xf) : out;
    AMDP_GEMM(gemm32(kt, T, h, d_.ffn, F(A.f), d_.ffn, false, W + P.fc2.off, d_.ffn, false, nx, h, AMDP_EPI_RESIDUAL, s,
                     F(A.hmid), h), 1);
    x = nx;
  }
  if (last()) {
    wait_seg();
    AMDP_TRY(K_LAYERNORM, 0, 8.0 * T * h, amdp_f32_layernorm_fwd(F(a.xf), W + lnf_g_.off, W + lnf_b_.off, F(a.lnf),
                                                                a.lnf_mean, a.lnf_rstd, T, h, d_.ln_eps, st), 1);
    AMDP_GEMM(gemm32(kt, T, d_.V, h, F(a.lnf), h, false, W + head_.off, h, false, F(a.logits), d_.V, AMDP_EPI_STORE_F32, s), 1);
    AMDP_TRY(K_XENT, 0, 12.0 * T * d_.V, amdp_f32_xent_fwd_bwd(F(a.logits), labels, loss_sum, ws.rows, T, d_.V, d_.V,
                                                               loss_scale, st), 2);
  }
  return launched;
}

int GptStage::backward_f32(const SlotActs& a, const int32_t* tokens, const float* in, const float* gin, float* gout,
                           uint8_t* wsb, cudaStream_t s, int* rc, const int32_t* key_len) const {
  int launched = 0;
  *rc = 0;
  auto st = reinterpret_cast<amdp_stream_t>(s);
  const int T = d_.T, h = d_.h, Fn = d_.ffn;
  const Ws ws = carve_ws(d_, wsb);
  const float* W = master;
  float *g0 = F(ws.g0), *g1 = F(ws.g1), *dU = F(ws.dU), *dqkv = F(ws.dqkv), *dtmp = F(ws.dtmp), *dh = F(ws.dhmid);
  const float* g = gin;
  if (last()) {  // logits hold dloss/dlogits (written by the forward's cross-entropy)
    AMDP_GEMM(gemm32(kt, d_.V, h, T, F(a.logits), d_.V, true, F(a.lnf), h, true, grad + head_.off, h, AMDP_EPI_ACCUM_F32, s), 1);
    AMDP_GEMM(gemm32(kt, T, h, d_.V, F(a.logits), d_.V, false, W + head_.off, h, true, dtmp, h, AMDP_EPI_STORE_F32, s), 1);
    AMDP_TRY(K_LAYERNORM, 0, 16.0 * T * h, amdp_f32_layernorm_bwd(dtmp, F(a.xf), W + lnf_g_.off, a.lnf_mean, a.lnf_rstd,
                                                                 nullptr, g0, grad + lnf_g_.off, grad + lnf_b_.off, T, h, st), 2);
    g = g0;
  }
  for (int li = l1_ - l0_ - 1; li >= 0; --li) {
    const LayerParams& P = layers_[static_cast<size_t>(li)];
    const LayerActs& A = a.layers[static_cast<size_t>(li)];
    const float* x = li > 0 ? F(A.x) : (first() ? F(a.x0) : in);
    // y = hmid + f W2^T
    AMDP_GEMM(gemm32(kt, h, Fn, T, g, h, true, F(A.f), Fn, true, grad + P.fc2.off, Fn, AMDP_EPI_ACCUM_F32, s), 1);
    AMDP_GEMM(gemm32(kt, T, Fn, h, g, h, false, W + P.fc2.off, Fn, true, dU, Fn, AMDP_EPI_GELU_BWD, s, F(A.u), Fn), 1);
    // f = gelu(ln2 W1^T)
    AMDP_GEMM(gemm32(kt, Fn, h, T, dU, Fn, true, F(A.ln2), h, true, grad + P.fc1.off, h, AMDP_EPI_ACCUM_F32, s), 1);
    AMDP_GEMM(gemm32(kt, T, h, Fn, dU, Fn, false, W + P.fc1.off, h, true, dtmp, h, AMDP_EPI_STORE_F32, s), 1);
    AMDP_TRY(K_LAYERNORM, 0, 16.0 * T * h, amdp_f32_layernorm_bwd(dtmp, F(A.hmid), W + P.ln2_g.off, A.ln2_mean, A.ln2_rstd, g,
                                                                 dh, grad + P.ln2_g.off, grad + P.ln2_b.off, T, h, st), 2);
    // hmid = x + o Wo^T
    AMDP_GEMM(gemm32(kt, h, h, T, dh, h, true, F(A.o), h, true, grad + P.o.off, h, AMDP_EPI_ACCUM_F32, s), 1);
    AMDP_GEMM(gemm32(kt, T, h, h, dh, h, false, W + P.o.off, h, true, dtmp, h, AMDP_EPI_STORE_F32, s), 1);
    AMDP_TRY(K_ATTN_BWD, 2.5 * attn_fwd_flops(), 0, amdp_f32_attention_bwd(F(A.qkv), F(A.o), dtmp, A.lse, dqkv, ws.attn, d_.B,
                                                                           d_.S, d_.heads, d_.hd, d_.causal ? 1 : 0, key_len, st), 3);
    // qkv = ln1 Wqkv^T
    AMDP_GEMM(gemm32(kt, 3 * h, h, T, dqkv, 3 * h, true, F(A.ln1), h, true, grad + P.qkv.off, h, AMDP_EPI_ACCUM_F32, s), 1);
    AMDP_GEMM(gemm32(kt, T, h, 3 * h, dqkv, 3 * h, false, W + P.qkv.off, h, true, dtmp, h, AMDP_EPI_STORE_F32, s), 1);
    float* gn = (li == 0 && !first()) ? gout : (g == g0 ? g1 : g0);
    AMDP_TRY(K_LAYERNORM, 0, 16.0 * T * h, amdp_f32_layernorm_bwd(dtmp, x, W + P.ln1_g.off, A.ln1_mean, A.ln1_rstd, dh, gn,
                                                                 grad + P.ln1_g.off, grad + P.ln1_b.off, T, h, st), 2);
    g = gn;
  }
  if (first())
    AMDP_TRY(K_EMBED, 0, 20.0 * T * h, amdp_f32_embedding_bwd(tokens, g, grad + wte_.off, grad + wpe_.off, ws.rows, T, d_.S,
                                                              h, st), 3);
  return launched;
}

}  // namespace amdp
