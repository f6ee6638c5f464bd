// nurbs_kernels.cu — the non-grid kernels of the NURBS-Diff hot path (arXiv 2104.14547):
// fixed-order cross-tile reduction, span/basis tables, checked-mode validation,
// and the launch dispatch to the per-degree grid kernels (nurbs_grid.cuh).
// Citations: P:n = reference/PAPER.md line n; R<k> = reading k of DESIGN.md §3.
#include <cuda_runtime.h>
#include <cstdint>

#include "nurbs_device.cuh"

namespace nb {

// ------------------------------------------------------------------------ cross-tile reduce
// dQ_ij = sum over row blocks rb (ascending) and column blocks cb (ascending) whose bands
// contain (i, j) of the tile partials; then the Eq.8/9 epilogue. One thread per control point.
template <bool FIT>
__global__ void __launch_bounds__(256) nurbs_reduce_kernel(const Params prm, int P) {
  const long long total = (long long)prm.B * prm.r.n * prm.c.n;
  const long long gsz = (long long)gridDim.x * blockDim.x;
  const long long idx0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (prm.gR)
    for (long long x = idx0; x < (long long)prm.gR_items * prm.gR_per; x += gsz) prm.gR[x] = 0.f;
  if (prm.gC)
    for (long long x = idx0; x < (long long)prm.gC_items * prm.gC_per; x += gsz) prm.gC[x] = 0.f;
  if (FIT && blockIdx.x == 0 && threadIdx.x < 32) {  // loss = mean |S - T|^2, fixed order
    float a = 0.f;
    for (int x = threadIdx.x; x < prm.n_parts; x += 32) a += prm.loss_parts[x];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (threadIdx.x == 0) *prm.loss = a * (0.5f * prm.fit_scale);
  }
  for (long long idx = idx0; idx < total; idx += gsz) {
    const float4 c = __ldg(prm.ctrl + idx);
    float4 g;
    if (FIT && prm.direct) {
      g = prm.gctrl[idx];  // written by the grid kernel's epilogue
    } else {
      const int m = prm.c.n;
      const int j = (int)(idx % m);
      const long long t2 = idx / m;
      const int i = (int)(t2 % prm.r.n);
      const int s = (int)(t2 / prm.r.n);
      const int K = prm.K;
      const int rb_hi = min(prm.NRB - 1, i / K);
      const int x = i - K - P + 1;
      const int rb_lo = x <= 0 ? 0 : (x + K - 1) / K;
      const int2* cbands = prm.colband + (size_t)s * prm.NCB;
      int lo = 0, hi = prm.NCB;  // first cb with j1 >= j
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cbands[mid].y < j) lo = mid + 1; else hi = mid;
      }
      int cb_hi = lo;  // one past the last column block whose band contains j
      while (cb_hi < prm.NCB && cbands[cb_hi].x <= j) ++cb_hi;
      const int nrb = rb_hi - rb_lo + 1, ncb = cb_hi - lo;
      const float4* sl = prm.slots + (((size_t)s * prm.NRB) * prm.NCB) * prm.T_rows * m + j;
      auto slot = [&](int rb, int cb) {
        return sl + (((size_t)rb * prm.NCB + cb) * prm.T_rows + (i - rb * K)) * m;
      };
      float4 a4 = f4(0.f);
      constexpr int RBX = kMaxQ + 1, CBX = 2;  // the common case: every load issued before the sums
      if (nrb <= RBX && ncb <= CBX) {
        float4 v[RBX][CBX];
#pragma unroll
        for (int u = 0; u < RBX; ++u)
#pragma unroll
          for (int w = 0; w < CBX; ++w) v[u][w] = (u < nrb && w < ncb) ? *slot(rb_lo + u, lo + w) : f4(0.f);
#pragma unroll
        for (int u = 0; u < RBX; ++u)  // rb ascending, then cb ascending (the fixed order)
#pragma unroll
          for (int w = 0; w < CBX; ++w)
            if (u < nrb && w < ncb) {
              a4.x += v[u][w].x; a4.y += v[u][w].y; a4.z += v[u][w].z; a4.w += v[u][w].w;
            }
      } else {
        for (int rb = rb_lo; rb <= rb_hi; ++rb)
          for (int cb = lo; cb < cb_hi; ++cb) {
            const float4 v = *slot(rb, cb);
            a4.x += v.x; a4.y += v.y; a4.z += v.z; a4.w += v.w;
          }
      }
      // epilogue (Eq.8/9): dP = w dQ_xyz, dw = P.dQ_xyz + dQ_w
      g = make_float4(c.w * a4.x, c.w * a4.y, c.w * a4.z, fmaf(c.x, a4.x, fmaf(c.y, a4.y, fmaf(c.z, a4.z, a4.w))));
      if (prm.gctrl) prm.gctrl[idx] = g;
    }
    if (FIT)  // SGD step (Eq.14): Psi <- Psi - lr dL/dPsi on P and w
      prm.ctrl_mut[idx] = make_float4(fmaf(-prm.lr, g.x, c.x), fmaf(-prm.lr, g.y, c.y), fmaf(-prm.lr, g.z, c.z),
                                      fmaf(-prm.lr, g.w, c.w));
  }
}

// ------------------------------------------------------------------------ tables
__global__ void nurbs_tables_kernel(Dir R, Dir C, unsigned char* tab, TabLayout L) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx == 0) {
    int* h = reinterpret_cast<int*>(tab);
    h[0] = (int)kTabMagic; h[1] = 1;
    h[2] = R.n; h[3] = R.p; h[4] = R.ns; h[5] = L.np_r;
    h[6] = C.n; h[7] = C.p; h[8] = C.ns; h[9] = L.np_c;
  }
  const Dir& D = idx < R.ns ? R : C;
  const int a = idx < R.ns ? idx : idx - R.ns;
  if (idx >= R.ns + C.ns) return;
  int* span = reinterpret_cast<int*>(tab + (idx < R.ns ? L.off_span_r : L.off_span_c));
  float* N = reinterpret_cast<float*>(tab + (idx < R.ns ? L.off_N_r : L.off_N_c));
  const int np = idx < R.ns ? L.np_r : L.np_c;
  const float x = __ldg(D.s + a);
  float nb_[kMaxQ + 1];
  int sp = 0;
  if (D.p == 0) {
    nb_[0] = 1.f;
  } else {
    sp = d_find_span(D.knots, D.n, D.p, x);
    d_basis<kMaxQ>(D.knots, sp, x, D.p, nb_);
  }
  span[a] = sp;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (k < np) N[(size_t)a * np + k] = (k <= D.p && k <= kMaxQ) ? nb_[k <= kMaxQ ? k : 0] : 0.f;
  if (idx < R.ns && L.nsf_r > 0) {  // sfirst[s - p] = a for the spans s in (span(a-1), span(a)]
    int* sf = reinterpret_cast<int*>(tab + L.off_sfirst_r);
    const int prev = a > 0 ? d_find_span(D.knots, D.n, D.p, __ldg(D.s + a - 1)) : D.p - 1;
    for (int k = max(prev + 1, D.p); k <= min(sp, D.n); ++k) sf[k - D.p] = a;
    if (a == R.ns - 1)  // spans past the last sample's
      for (int k = max(sp + 1, D.p); k <= D.n; ++k) sf[k - D.p] = R.ns;
  }
}

// ------------------------------------------------------------------------ validation
// status = min over violations of (code << 48 | which << 40 | index).
__device__ __forceinline__ void report(unsigned long long* st, int code, int which, long long index) {
  const unsigned long long key =
      ((unsigned long long)code << 48) | ((unsigned long long)which << 40) | ((unsigned long long)index & 0xffffffffffull);
  atomicMin(st, key);
}

__global__ void nurbs_validate_kernel(int B, Dir R, Dir C, int check_rows, const float4* ctrl, long long n_ctrl,
                                      unsigned long long* st) {
  const long long gsz = (long long)gridDim.x * blockDim.x;
  const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int items_r = R.kstride ? B : 1, items_c = C.kstride ? B : 1;
  // weights and finiteness (code 5 = NURBS_E_WEIGHT), which = 0
  for (long long x = i0; x < n_ctrl; x += gsz) {
    const float4 c = ctrl[x];
    if (!(c.w > 0.f) || !isfinite(c.w) || !isfinite(c.x) || !isfinite(c.y) || !isfinite(c.z)) report(st, 5, 0, x);
  }
  for (int d = 0; d < 2; ++d) {
    const Dir& D = d == 0 ? R : C;
    if (d == 0 && !check_rows) continue;
    const int items = d == 0 ? items_r : items_c;
    const int nk = D.n + D.p + 1;
    // knots non-decreasing, finite, non-empty domain (code 3 = NURBS_E_KNOTS), which = 1 + d
    for (long long x = i0; x < (long long)items * nk; x += gsz) {
      const int it = (int)(x / nk), k = (int)(x % nk);
      const float* Uk = D.knots + (long long)it * D.kstride;
      if (!isfinite(Uk[k])) report(st, 3, 1 + d, x);
      if (k + 1 < nk && !(Uk[k] <= Uk[k + 1])) report(st, 3, 1 + d, x);
      if (k == 0 && !(Uk[D.p] < Uk[D.n])) report(st, 3, 1 + d, x);
    }
    // samples sorted (code 6) and inside every item's domain (code 4), which = 3 + d
    for (long long x = i0; x < (long long)items * D.ns; x += gsz) {
      const int it = (int)(x / D.ns), a = (int)(x % D.ns);
      const float* Uk = D.knots + (long long)it * D.kstride;
      const float u = D.s[a];
      if (it == 0 && a + 1 < D.ns && !(u <= D.s[a + 1])) report(st, 6, 3 + d, a);
      if (!(u >= Uk[D.p] && u <= Uk[D.n])) report(st, 4, 3 + d, a);
    }
  }
}

// ------------------------------------------------------------------------ launchers
size_t grid_smem_bytes(bool bwd, int P, int q, int T_rows, int CBW, int kg, bool tmap) {
  const int NP = (P + 1) <= 4 ? 4 : 8;
  const int NQ = (q + 1) <= 4 ? 4 : 8;
  const int rps = bwd ? kRPS_B : kRPS_F, nst = bwd ? (kg != 0 ? 2 : kStages_B) : kStages_F;
  const int nrt = tmap && P > 0 && !bwd ? 2 : 1;  // row tables double-buffered (tensor-map forward)
  size_t b = (((size_t)T_rows * CBW * 16 + 127) & ~(size_t)127) + (size_t)nst * rps * kCB * 3 * 4 + nrt * kRowChunk * 4 +
             (size_t)nrt * kRowChunk * NP * 4;
  if (bwd) b += (size_t)kHRing * kCB * 16 + kCB * 4 + (size_t)kCB * NQ * 4 + (kCB + 4) * 4;
  b += 4 * 4;                                  // misc
  b = (b + 7) / 8 * 8 + (1 + 2 * nst) * 8 + nst * 4;  // mbarriers + stage counters
  if (kg == 1)  // rowdot + the per-warp stage buffers of the row dot products (NEXT-4)
    b += 16 + (size_t)(kThreads / 32) * kRowChunk * (P + 1) * 4 + (size_t)(kThreads / 32) * 4 * (P + 1) * 36 * 4;
  if (kg == 2) {  // span moments (NEXT-4): per-warp lane rows [4][32][KXS] + span sums [4][kRMax][KNX]
    const int knx = (P + 1) * (P + 1), kxs = knx | 1;
    b += 16 + (size_t)(kThreads / 32) * 32 * kxs * 4 + (size_t)(kThreads / 32) * kRMax * knx * 4;
  }
  return b;
}

cudaError_t launch_grid(const Params& prm, int mode, int P, int q, cudaStream_t st) {
  switch (P) {
    case 0: return launch_grid_p0(prm, mode, q, st);
    case 1: return launch_grid_p1(prm, mode, q, st);
    case 2: return launch_grid_p2(prm, mode, q, st);
    case 3: return launch_grid_p3(prm, mode, q, st);
    case 4: return launch_grid_p4(prm, mode, q, st);
    case 5: return launch_grid_p5(prm, mode, q, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_reduce(const Params& prm, int P, cudaStream_t st) {
  const long long total = (long long)prm.B * prm.r.n * prm.c.n;
  long long blocks = (total + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 32) blocks = 148 * 32;
  nurbs_reduce_kernel<false><<<(unsigned)blocks, 256, 0, st>>>(prm, P);
  return cudaGetLastError();
}

cudaError_t launch_fit_update(const Params& prm, int P, cudaStream_t st) {
  const long long total = (long long)prm.B * prm.r.n * prm.c.n;
  long long blocks = (total + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 32) blocks = 148 * 32;
  nurbs_reduce_kernel<true><<<(unsigned)blocks, 256, 0, st>>>(prm, P);
  return cudaGetLastError();
}

cudaError_t launch_tables(const Dir& r, const Dir& c, void* tables, const TabLayout& L, cudaStream_t st) {
  const int total = r.ns + c.ns;
  const int blocks = total > 0 ? (total + 255) / 256 : 1;
  nurbs_tables_kernel<<<blocks, 256, 0, st>>>(r, c, static_cast<unsigned char*>(tables), L);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------ ordered partial sum
// out[k] = sum over parts r = 0, 1, ... (ascending) of parts[r][k] (multi-GPU point sharding:
// the rank partials of the backward, after an all-gather). float4 when n % 4 == 0.
__global__ void __launch_bounds__(256) nurbs_sum_partials_kernel(const float* __restrict__ parts, int np, long long n,
                                                                 float* out) {
  const long long gsz = (long long)gridDim.x * blockDim.x;
  const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if ((n & 3) == 0) {
    const long long n4 = n >> 2;
    const float4* p4 = reinterpret_cast<const float4*>(parts);
    for (long long i = i0; i < n4; i += gsz) {
      float4 a = __ldg(p4 + i);
      for (int r = 1; r < np; ++r) {
        const float4 b = __ldg(p4 + (long long)r * n4 + i);
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
      }
      reinterpret_cast<float4*>(out)[i] = a;
    }
  } else {
    for (long long i = i0; i < n; i += gsz) {
      float a = __ldg(parts + i);
      for (int r = 1; r < np; ++r) a += __ldg(parts + (long long)r * n + i);
      out[i] = a;
    }
  }
}

cudaError_t launch_sum_partials(const float* parts, int np, long long n, float* out, cudaStream_t st) {
  const long long work = (n & 3) == 0 ? n / 4 : n;
  long long blocks = (work + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  nurbs_sum_partials_kernel<<<(unsigned)blocks, 256, 0, st>>>(parts, np, n, out);
  return cudaGetLastError();
}

cudaError_t launch_validate(int B, const Dir& r, const Dir& c, int check_rows, const float4* ctrl,
                            long long n_ctrl, unsigned long long* status, cudaStream_t st) {
  nurbs_validate_kernel<<<148 * 4, 256, 0, st>>>(B, r, c, check_rows, ctrl, n_ctrl, status);
  return cudaGetLastError();
}

}  // namespace nb
