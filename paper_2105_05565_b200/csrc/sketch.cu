// a1 -- sketch draw.  One CTA of 1024 threads regenerates the sketch of
// iteration k from (seed, k) with Philox4x32-10 and writes it in bucket order.
//
//  Subsample (Eq. subsample) / SubCount selection:
//    key64_i = (x << 32) | y of Philox((i, k, 0, 0), key); the selected set is the L indices with the
//    smallest (key64_i, i).  Found by an 8-pass, 8-bit-digit radix select of the L-th smallest key
//    (histograms in shared memory), then compaction and a bitonic sort of the L survivors by
//    (key64, i).  SubCount: position j -> bucket j / k, sign 1 - 2 (x & 1) of Philox((c_j, k, 2, 0)).
//  Count: h(i) = floor(x tau / 2^32), sign 1 - 2 (y & 1) of Philox((i, k, 1, 0)); the
//    entries are placed in bucket order, ascending coordinate inside a bucket, deterministically:
//    per-warp bucket histograms -> offsets -> warp-ordered placement with __match_any_sync ranks.
#include "rs_internal.cuh"

namespace rs {

namespace {

constexpr int kThreads = 1024;
constexpr int kMaxSelect = 8192;      // largest L the single-CTA select+sort handles
constexpr int kKeyCache = 8192;       // keys kept in shared memory when m <= kKeyCache
constexpr int kMaxCountTau = 1536;    // per-warp histograms 32 x tau ints in shared memory

__device__ __forceinline__ unsigned long long sel_key(unsigned i, unsigned it, uint2 key) {
  uint4 o = philox4x32_10(make_uint4(i, it, STREAM_SELECT, 0u), key);
  return ((unsigned long long)o.x << 32) | o.y;
}

__device__ __forceinline__ bool lt_pair(unsigned long long ka, unsigned ia, unsigned long long kb,
                                        unsigned ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__global__ void __launch_bounds__(kThreads, 1)
k_sketch_select(DevSketch skb, uint2 key, const Ctrl* ctrl, long long fixed_k, long long kofs,
                int* err) {
  if (fixed_k < 0 && slot_unused(ctrl, kofs + blockIdx.x)) return;
  // slot blockIdx.x of a batch receives the sketch of iteration k0 + blockIdx.x
  const DevSketch sk = skb.at(blockIdx.x);
  const unsigned it = (unsigned)((fixed_k >= 0 ? fixed_k : ctrl->k + kofs) + blockIdx.x);
  const int m = sk.m, L = sk.len, tid = threadIdx.x;
  extern __shared__ unsigned long long dsm[];
  // layout: [cache: kc u64][sort keys: Lp u64][sort idx: Lp u32]
  const int kc = m <= kKeyCache ? m : 0;
  int Lp = 1;
  while (Lp < L) Lp <<= 1;
  unsigned long long* cache = dsm;
  unsigned long long* skey = dsm + kc;
  unsigned* sidx = reinterpret_cast<unsigned*>(skey + Lp);

  __shared__ unsigned hist[256];
  __shared__ unsigned long long s_prefix, s_mask;
  __shared__ unsigned s_remaining, s_neq, s_eqcount, s_lesscount;
  __shared__ unsigned s_eq[1024];

  for (int i = tid; i < kc; i += kThreads) cache[i] = sel_key(i, it, key);
  if (tid == 0) { s_prefix = 0; s_mask = 0; s_remaining = L; }
  __syncthreads();

  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = tid; b < 256; b += kThreads) hist[b] = 0;
    __syncthreads();
    const unsigned long long pre = s_prefix, msk = s_mask;
    for (int i = tid; i < m; i += kThreads) {
      const unsigned long long kk = kc ? cache[i] : sel_key(i, it, key);
      if ((kk & msk) == pre) atomicAdd(&hist[(kk >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l owns bins [8l, 8l+8)
      unsigned loc[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) { loc[q] = hist[tid * 8 + q]; sum += loc[q]; }
      unsigned incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += v;
      }
      const unsigned excl = incl - sum, rem = s_remaining;
      if (excl < rem && rem <= incl) {
        unsigned c = excl;
        int dsel = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (c < rem && rem <= c + loc[q]) { dsel = q; break; }
          c += loc[q];
        }
        const unsigned digit = tid * 8 + dsel;
        s_remaining = rem - c;
        s_prefix = pre | ((unsigned long long)digit << shift);
        s_mask = msk | (255ull << shift);
        if (shift == 0) s_neq = loc[dsel];
      }
    }
    __syncthreads();
  }
  const unsigned long long T = s_prefix;
  const unsigned need_eq = s_remaining;           // >= 1
  const unsigned n_less = (unsigned)L - need_eq;
  const unsigned n_eq = s_neq;
  if (tid == 0) { s_lesscount = 0; s_eqcount = 0; }
  __syncthreads();
  if (n_eq > 1024) {   // astronomically unlikely with 64-bit Philox keys: fail the solve loudly
    if (tid == 0) {
      if (ctrl) {
        Ctrl* c = const_cast<Ctrl*>(ctrl);
        c->status = ST_SKETCHFAIL;
        c->done = 1;
      } else {
        atomicExch(err, 1);   // rs_sketch_draw reads and clears it
      }
    }
    return;
  }
  for (int i = tid; i < m; i += kThreads) {
    const unsigned long long kk = kc ? cache[i] : sel_key(i, it, key);
    if (kk < T) {
      const unsigned p = atomicAdd(&s_lesscount, 1u);
      skey[p] = kk;
      sidx[p] = i;
    } else if (kk == T) {
      const unsigned p = atomicAdd(&s_eqcount, 1u);
      s_eq[p] = i;
    }
  }
  __syncthreads();
  // keys equal to T: keep the need_eq smallest indices (tie rule (key64, i))
  for (unsigned q = tid; q < n_eq; q += kThreads) {
    const unsigned iq = s_eq[q];
    unsigned rank = 0;
    for (unsigned t = 0; t < n_eq; ++t) rank += s_eq[t] < iq;
    if (rank < need_eq) { skey[n_less + rank] = T; sidx[n_less + rank] = iq; }
  }
  for (int p = L + tid; p < Lp; p += kThreads) { skey[p] = ~0ull; sidx[p] = 0xffffffffu; }
  __syncthreads();
  // bitonic sort of Lp (key, idx) pairs ascending
  for (int size = 2; size <= Lp; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = tid; t < (Lp >> 1); t += kThreads) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long ka = skey[lo], kb = skey[hi];
        const unsigned ia = sidx[lo], ib = sidx[hi];
        const bool swap = up ? lt_pair(kb, ib, ka, ia) : lt_pair(ka, ia, kb, ib);
        if (swap) { skey[lo] = kb; skey[hi] = ka; sidx[lo] = ib; sidx[hi] = ia; }
      }
      __syncthreads();
    }
  }
  const int ks = sk.kind == SK_SUBCOUNT ? sk.ksum : 1;
  for (int j = tid; j < L; j += kThreads) {
    const unsigned c = sidx[j];
    sk.coord[j] = (int)c;
    sk.bucket[j] = j / ks;
    signed char sg = 1;
    if (sk.kind == SK_SUBCOUNT) {
      uint4 o = philox4x32_10(make_uint4(c, it, STREAM_SUBCOUNT_SIGN, 0u), key);
      sg = (o.x & 1u) ? -1 : 1;
    }
    sk.sign[j] = sg;
  }
  for (int b = tid; b <= sk.tau; b += kThreads) sk.bptr[b] = b * ks;
}

__global__ void __launch_bounds__(kThreads, 1)
k_sketch_count(DevSketch skb, uint2 key, const Ctrl* ctrl, long long fixed_k, long long kofs) {
  if (fixed_k < 0 && slot_unused(ctrl, kofs + blockIdx.x)) return;
  const DevSketch sk = skb.at(blockIdx.x);
  const unsigned it = (unsigned)((fixed_k >= 0 ? fixed_k : ctrl->k + kofs) + blockIdx.x);
  const int m = sk.m, tau = sk.tau, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  extern __shared__ unsigned long long dsm[];
  unsigned* hist = reinterpret_cast<unsigned*>(dsm);   // [32][tau]
  __shared__ unsigned s_tot[kThreads];
  for (int q = tid; q < 32 * tau; q += kThreads) hist[q] = 0;
  __syncthreads();
  const int seg = (m + 31) / 32;
  const int beg = warp * seg, end = min(m, beg + seg);
  // Phase A: hash every coordinate of the warp's segment; per-warp bucket counts.
  for (int i = beg + lane; i < end; i += 32) {
    uint4 o = philox4x32_10(make_uint4((unsigned)i, it, STREAM_COUNT, 0u), key);
    const unsigned h = __umulhi(o.x, (unsigned)tau);       // floor(x * tau / 2^32)
    sk.cmap[i] = (int)((h << 1) | (o.y & 1u));
    atomicAdd(&hist[warp * tau + h], 1u);
  }
  __syncthreads();
  // Phase B: bucket totals, exclusive scan -> bptr, per-(warp, bucket) offsets.
  // thread t owns buckets [t*per, (t+1)*per)
  const int per = (tau + kThreads - 1) / kThreads;
  unsigned tsum = 0;
  for (int q = 0; q < per; ++q) {
    const int b = tid * per + q;
    if (b < tau) {
      unsigned c = 0;
      for (int w = 0; w < 32; ++w) c += hist[w * tau + b];
      tsum += c;
    }
  }
  s_tot[tid] = tsum;
  __syncthreads();
  for (int o = 1; o < kThreads; o <<= 1) {  // Hillis-Steele inclusive scan
    unsigned v = tid >= o ? s_tot[tid - o] : 0u;
    __syncthreads();
    s_tot[tid] += v;
    __syncthreads();
  }
  unsigned run = s_tot[tid] - tsum;
  for (int q = 0; q < per; ++q) {
    const int b = tid * per + q;
    if (b < tau) {
      sk.bptr[b] = (int)run;
      for (int w = 0; w < 32; ++w) {
        const unsigned c = hist[w * tau + b];
        hist[w * tau + b] = run;
        run += c;
      }
    }
  }
  if (tid == 0) sk.bptr[tau] = m;
  __syncthreads();
  // Phase C: warp-ordered placement (ascending coordinate within each bucket).
  for (int base = beg; base < end; base += 32) {
    const int i = base + lane;
    const bool act = i < end;
    const unsigned amask = __ballot_sync(0xffffffffu, act);
    if (act) {
      const unsigned cm = (unsigned)sk.cmap[i];
      const unsigned b = cm >> 1;
      const unsigned peers = __match_any_sync(amask, b);
      const unsigned rank = __popc(peers & ((1u << lane) - 1u));
      const unsigned pos = hist[warp * tau + b] + rank;
      sk.coord[pos] = i;
      sk.bucket[pos] = (int)b;
      sk.sign[pos] = (cm & 1u) ? -1 : 1;
      __syncwarp(amask);
      if (rank == 0) hist[warp * tau + b] += __popc(peers);
    }
    __syncwarp();
  }
}

}  // namespace

size_t sketch_max_len(int kind, int m, int tau, int ksum) {
  if (kind == SK_SUBSAMPLE) return (size_t)tau;
  if (kind == SK_SUBCOUNT) return (size_t)tau * (size_t)ksum;
  return (size_t)m;
}

static int* g_err_flag = nullptr;   // device int set if the select hits an unsupported tie storm

// One-time, per-device setup (never inside a stream capture): kernel attributes, error flag.
cudaError_t sketch_init() {
  cudaError_t e = cudaFuncSetAttribute(k_sketch_count, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       32 * kMaxCountTau * (int)sizeof(unsigned));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_sketch_select, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kKeyCache * 8 + kMaxSelect * 12);
  if (e != cudaSuccess) return e;
  if (!g_err_flag) {
    e = cudaMalloc(&g_err_flag, sizeof(int));
    if (e != cudaSuccess) return e;
    e = cudaMemset(g_err_flag, 0, sizeof(int));
  }
  return e;
}

cudaError_t sketch_err_take(int* out) {
  *out = 0;
  if (!g_err_flag) return cudaSuccess;
  cudaError_t e = cudaMemcpy(out, g_err_flag, sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && *out) e = cudaMemset(g_err_flag, 0, sizeof(int));
  return e;
}

cudaError_t launch_sketch(const DevSketch& sk, uint64_t seed, const Ctrl* ctrl, long long fixed_k,
                          cudaStream_t st) {
  return launch_sketch_batch(sk, 1, seed, ctrl, fixed_k, st, 0);
}

cudaError_t launch_sketch_batch(const DevSketch& sk, int nslots, uint64_t seed, const Ctrl* ctrl,
                                long long fixed_k, cudaStream_t st, long long kofs) {
  if (nslots < 1) return cudaErrorInvalidValue;
  const uint2 key = make_uint2((unsigned)(seed & 0xffffffffull), (unsigned)(seed >> 32));
  if (sk.kind == SK_COUNT) {
    if (sk.tau > kMaxCountTau) return cudaErrorInvalidValue;
    const size_t smem = (size_t)32 * sk.tau * sizeof(unsigned);
    k_sketch_count<<<nslots, kThreads, smem, st>>>(sk, key, ctrl, fixed_k, kofs);
    return cudaGetLastError();
  }
  if (sk.len > kMaxSelect) return cudaErrorInvalidValue;
  if (!g_err_flag) return cudaErrorInitializationError;   // sketch_init() not called
  int Lp = 1;
  while (Lp < sk.len) Lp <<= 1;
  const int kc = sk.m <= kKeyCache ? sk.m : 0;
  const size_t smem = (size_t)kc * 8 + (size_t)Lp * 12;
  k_sketch_select<<<nslots, kThreads, smem, st>>>(sk, key, ctrl, fixed_k, kofs, g_err_flag);
  return cudaGetLastError();
}

}  // namespace rs
