// nurbs_bwd_tc.cu — the grid backward of the NURBS-Diff hot path on the 5th-generation tensor
// cores (tcgen05 + TMEM), for control nets of at most 32 columns.
//
// Citations: P:n = reference/PAPER.md line n; R<k> = reading k of DESIGN.md §3.
//
// The backward (Eq.8, Eq.9, J^T g of P:251) on one tile (surface s,
// row block, 128-sample column block; the same plan as the SIMT grid kernel) is
//   S'[a][b] = sum_i sum_j Nu[a][i] Nv[b][j] Q[i][j]          (recompute, Eq.3 homogeneous)
//   G[a][b]  = (g/W, -(g.S)/W)                                 (per point, W = S'_w)
//   dQ[i][j] = sum_a sum_b Nu[a][i] Nv[b][j] G[a][b]           (Alg.2)
// with dP = w dQ_xyz, dw = P.dQ_xyz + dQ_w. Thread / TMEM lane b owns one sample column.
// Per chunk of R = 8 sample rows a:
//   X  [a,c][j] = sum_r Nu[a][r] Q[su(a)-p+r][j][c]           SIMT (p+1 taps), -> smem (B operand)
//   MMA1  D1[b][(a,c)] = sum_j NvA[b][j] X[(a,c)][j]           tcgen05 M=128 N=32 K=16|32
//   G from D1 (TMEM -> registers) and g (TMA-staged)           SIMT, -> TMEM (A operand)
//   MMA2  D2_c[b][i] += sum_a G_c[b][a] Nu[a][i]               tcgen05 M=128 N=16 K=8, per c
// and once per tile B2: dQ[i][j] = sum_b Nv[b][j] H[b][i] with H = D2 (SIMT gather in
// ascending b). Both MMAs run as 3xTF32 (hi*hi + hi*lo + lo*hi, x = hi + lo), so products carry
// ~21 significant bits: fp32-level error, far inside R16's 1e-4. Every sum has a fixed order,
// so results are bitwise repeatable; they are not bitwise equal to the SIMT kernel's.
//
// Persistent CTAs (two per SM: 2 x 256 TMEM columns), 192 threads: warps 0-3 compute (TMEM lane
// quadrants 0-3), warp 4 the TMA producer (per tile: row range, band spans, the control band;
// then the dL/dS ring, running ahead across tiles), warp 5 issues the MMAs (one thread).
// The chunk counter runs across tiles; the per-chunk barriers alternate by its parity.
#include <cuda_runtime.h>

#include "nurbs_tc.cuh"

namespace nb {
namespace tc {

constexpr int R = 8;             // sample rows per chunk (= kRPS_B: one TMA stage / tensor box)
constexpr int NI = 16;           // control rows of a band (MMA2 N); the plan keeps K + p <= 16
constexpr int NSTG = 5;          // dL/dS ring stages (two CTAs per SM: 10 x 12 KB of loads in flight)
constexpr int NH = NI / 2;       // control rows of H staged in smem at once (B2 in two halves)
constexpr int kThr = 192;
constexpr int kTmemCols = 256;
// TMEM columns. KJ = 16 (nets of <= 16 columns): NvA hi/lo in 0-31, ONE D1 buffer (32-63), TWO G
// buffers (64-127, 128-191; hi then lo), D2 192-255. KJ = 32: NvA 0-63, two D1 buffers (64-127),
// one G buffer (128-191), D2. With two G buffers the compute warps never wait for MMA2 of the
// previous chunk; with one D1 buffer, MMA1(k+1) starts as soon as D1(k) has been read.
template <int KJ>
struct Tm {
  static constexpr int NvHi = 0, NvLo = KJ == 16 ? 16 : 32;
  static constexpr int D1 = KJ == 16 ? 32 : 64, D1B = KJ == 16 ? 1 : 2;
  static constexpr int G = KJ == 16 ? 64 : 128, GB = KJ == 16 ? 2 : 1;  // buffer = 64 columns (hi 32, lo 32)
  static constexpr int D2 = 192;
};
constexpr int kSRow = kCB * 3;           // floats of a staged sample row (bulk IO)
constexpr int kHRow = 3 * kBoxCols;      // floats of one half row (tensor-map IO)
static_assert(R == kRPS_B, "one chunk is one backward TMA stage");

struct TileInfo {
  int s, rb, cb, a_lo, nwalk, jlo, ncol, pad;
};

template <int KJ, int NQ>
struct Layout {
  static constexpr size_t gst = 0;                                           // [NSTG][R][kSRow]
  static constexpr size_t hs = gst + (size_t)NSTG * R * kSRow * 4;            // [128][NH] float4
  static constexpr size_t band = hs + (size_t)kCB * NH * 16;                  // [2][NI][KJ] float4
  static constexpr size_t bandh = band + (size_t)2 * NI * KJ * 16;            // [NI][KJ] float4 (homogeneous)
  static constexpr size_t xs = bandh + (size_t)NI * KJ * 16;                  // [2 buf][hi,lo][32][KJ]
  static constexpr size_t nus = xs + (size_t)2 * 2 * 32 * KJ * 4;             // [3 buf][hi,lo][16][8]
  static constexpr size_t sus = nus + (size_t)3 * 2 * NI * R * 4;             // [kRowChunk] int
  static constexpr size_t nus_tab = sus + (size_t)kRowChunk * 4;              // [kRowChunk][4]
  static constexpr size_t svs = nus_tab + (size_t)kRowChunk * 4 * 4;          // [128] int
  static constexpr size_t nvs = svs + (size_t)kCB * 4;                        // [128][NQ]
  static constexpr size_t jb = nvs + (size_t)kCB * NQ * 4;                    // [KJ] int2
  static constexpr size_t tinfo = jb + (size_t)KJ * 8;                        // [2] TileInfo
  static constexpr size_t misc = tinfo + 2 * sizeof(TileInfo);                // [4] int
  static constexpr size_t bars = misc + 16;                                   // mbarriers
  static constexpr size_t bytes = bars + 26 * 8;
};

// First a in [0, ns) of the (sorted) sample rows whose span is >= S (ns if none): one thread.
__device__ __forceinline__ int first_row_at_span(const Dir& Rr, const float* Uk, int s_end, int S, int P) {
  int lo = 0, hi = Rr.ns;
  if (!Rr.tspan && S > s_end) return Rr.ns;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const bool ge = Rr.tspan ? (__ldg(Rr.tspan + mid) >= S) : (__ldg(Rr.s + mid) >= __ldg(Uk + S));
    if (ge) hi = mid; else lo = mid + 1;
  }
  (void)P;
  return lo;
}

template <int P, int Q, int KJ, int IO>
__global__ void __launch_bounds__(kThr, 2) nurbs_bwd_tc_kernel(const __grid_constant__ Params prm, int ntiles) {
  constexpr int NQ = (Q + 1) <= 4 ? 4 : 8;
  using L = Layout<KJ, NQ>;
  static_assert(P >= 1 && P + 1 <= 4, "row taps staged as float4");
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Dir& Rr = prm.r;
  const Dir& C = prm.c;
  const int m = C.n;
  const int CBW = prm.CBW;

  float* stage = reinterpret_cast<float*>(smem + L::gst);
  float4* Hs = reinterpret_cast<float4*>(smem + L::hs);
  float4* band0 = reinterpret_cast<float4*>(smem + L::band);
  float4* bandh = reinterpret_cast<float4*>(smem + L::bandh);
  using TM = Tm<KJ>;
  unsigned char* Xs = smem + L::xs;
  unsigned char* Nus = smem + L::nus;
  int* su_s = reinterpret_cast<int*>(smem + L::sus);
  float* Nu_s = reinterpret_cast<float*>(smem + L::nus_tab);
  int* sv_s = reinterpret_cast<int*>(smem + L::svs);
  float* Nv_s = reinterpret_cast<float*>(smem + L::nvs);
  int2* jb = reinterpret_cast<int2*>(smem + L::jb);
  TileInfo* tinfo = reinterpret_cast<TileInfo*>(smem + L::tinfo);
  int* misc = reinterpret_cast<int*>(smem + L::misc);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::bars);
  uint64_t* band_full = bars;             // [2] tile info + control band landed (1 + tx)
  uint64_t* band_empty = bars + 2;        // [2] tile done with the band (4 compute warps + MMA warp)
  uint64_t* sfull = bars + 4;             // [NSTG] TMA stage landed (1 + tx)
  uint64_t* sempty = bars + 4 + NSTG;     // [NSTG] stage consumed (4 compute warps)
  // per-chunk barriers, two of each (chunk k uses [k & 1], phase parity (k >> 1) & 1): a
  // barrier's next phase then always needs a step the waiter takes after its wait, so a phase
  // can never complete twice before it is observed
  uint64_t* xfull = bars + 4 + 2 * NSTG;  // [2] X(k), Nu(k) staged in smem (4 warps)
  uint64_t* d1full = xfull + 2;           // [2] MMA1(k) done (commit)
  uint64_t* gfull = xfull + 4;            // [2] G(k) in TMEM (4 warps)
  uint64_t* m2done = xfull + 6;           // [2] MMA2(k) done (commit)
  uint64_t* d1free = xfull + 8;           // [2] D1(k) read by the compute warps (4 warps; one D1 buffer)

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(band_full + i, 1u);
      mbar_init(band_empty + i, 5u);
      mbar_init(xfull + i, 4u);
      mbar_init(d1full + i, 1u);
      mbar_init(gfull + i, 4u);
      mbar_init(m2done + i, 1u);
      mbar_init(d1free + i, 4u);
    }
    for (int i = 0; i < NSTG; ++i) {
      mbar_init(sfull + i, 1u);
      mbar_init(sempty + i, 4u);
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(reinterpret_cast<uint32_t*>(misc), kTmemCols);
    tmem_relinquish();
  }
  fence_before_sync();
  __syncthreads();  // barriers initialised, TMEM allocated
  fence_after_sync();
  const uint32_t tbase = static_cast<uint32_t>(misc[0]);

  if (warp == 4) {
    // ================================ TMA producer (one thread)
    if (lane == 0) {
      int kg = 0, it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int buf = it & 1;
        if (it >= 2) mbar_wait(band_empty + buf, ((it >> 1) - 1) & 1);
        int bid = tile;
        const int cb = bid % prm.NCB;
        bid /= prm.NCB;
        const int rb = bid % prm.NRB;
        const int s = bid / prm.NRB;
        const int B0 = cb * kCB, cols = min(kCB, C.ns - B0);
        const int S0 = P + rb * prm.K, S1 = min(S0 + prm.K, Rr.n);
        const int band_lo = S0 - P, band_rows = S1 - band_lo;
        const float* Uk = Rr.knots + (long long)s * Rr.kstride;
        const float* Vk = C.tspan ? nullptr : C.knots + (long long)s * C.kstride;
        int a_lo = 0, a_hi = Rr.ns;
        if (prm.NRB > 1) {
          int s_end = Rr.n - 1;  // last non-empty span (R3)
          if (!Rr.tspan)
            while (s_end > P && __ldg(Uk + s_end) == __ldg(Uk + s_end + 1)) --s_end;
          if (rb > 0) a_lo = first_row_at_span(Rr, Uk, s_end, S0, P);
          if (rb < prm.NRB - 1) a_hi = first_row_at_span(Rr, Uk, s_end, S1, P);
        }
        const int nwalk = max(0, a_hi - a_lo);
        auto cspan = [&](int bb) -> int {
          int sp = C.tspan ? __ldg(C.tspan + bb) : d_find_span(Vk, m, Q, __ldg(C.s + bb));
          return min(max(sp, Q), m - 1);
        };
        const int jlo = cspan(B0) - Q;
        const int ncol = max(cspan(B0 + cols - 1), jlo + Q) - jlo + 1;  // <= m <= KJ (host rule)
        tinfo[buf] = TileInfo{s, rb, cb, a_lo, nwalk, jlo, ncol, 0};
        // the control band rows [band_lo, S1) x columns [jlo, jlo + ncol)
        float4* band = band0 + buf * (NI * KJ);
        const float4* src = prm.ctrl + ((size_t)s * Rr.n + band_lo) * m + jlo;
        const uint32_t rowb = (uint32_t)ncol * 16u;
        mbar_arrive_expect_tx(band_full + buf, rowb * band_rows);
        if (ncol == m && ncol == CBW) {
          bulk_g2s(band, src, rowb * band_rows, band_full + buf);
        } else {
          for (int r = 0; r < band_rows; ++r) bulk_g2s(band + r * CBW, src + (size_t)r * m, rowb, band_full + buf);
        }
        // the dL/dS rows of the tile, R rows per stage
        const int nc = (nwalk + R - 1) / R;
        if constexpr (IO >= 1) {
          const uint32_t rowbytes = (uint32_t)cols * 12u;
          const bool one_copy = (cols == C.ns) && cols == kCB;
          const size_t grow = (size_t)C.ns * 3;
          const size_t g0 = (((size_t)s * Rr.ns + a_lo) * C.ns + B0) * 3;
          const int nh = cols > kBoxCols ? 2 : 1;
          const uint32_t hb0 = (uint32_t)min(cols, kBoxCols) * 12u, hb1 = (uint32_t)max(0, cols - kBoxCols) * 12u;
          const int ty0 = s * Rr.ns + a_lo;
          for (int k = 0; k < nc; ++k, ++kg) {
            const int slot = kg % NSTG;
            if (kg >= NSTG) mbar_wait(sempty + slot, ((kg / NSTG) - 1) & 1);
            const int nr = min(R, nwalk - k * R);
            float* buf_g = stage + slot * (R * kSRow);
            const float* gsrc = prm.gout + g0 + (size_t)k * R * grow;
            if constexpr (IO == 2) {
              if (nr == R) {
                mbar_arrive_expect_tx(sfull + slot, (uint32_t)nh * R * kHRow * 4u);
                for (int h = 0; h < nh; ++h)
                  tma_load_2d(buf_g + h * R * kHRow, &prm.io_map, 3 * (B0 + h * kBoxCols), ty0 + k * R, sfull + slot);
              } else {
                mbar_arrive_expect_tx(sfull + slot, (hb0 + hb1) * nr);
                for (int rr = 0; rr < nr; ++rr) {
                  bulk_g2s(buf_g + rr * kHRow, gsrc + (size_t)rr * grow, hb0, sfull + slot);
                  if (hb1) bulk_g2s(buf_g + R * kHRow + rr * kHRow, gsrc + (size_t)rr * grow + kHRow, hb1, sfull + slot);
                }
              }
            } else {
              mbar_arrive_expect_tx(sfull + slot, rowbytes * nr);
              if (one_copy) {
                bulk_g2s(buf_g, gsrc, rowbytes * nr, sfull + slot);
              } else {
                for (int rr = 0; rr < nr; ++rr)
                  bulk_g2s(buf_g + rr * kSRow, gsrc + (size_t)rr * grow, rowbytes, sfull + slot);
              }
            }
          }
        }
      }
    }
  } else if (warp == 5) {
    // ================================ MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t id1 = idesc_tf32(128, 4 * R), id2 = idesc_tf32(128, NI);
      const uint64_t xd0 = sdesc(Xs, 128, (KJ / 4) * 128);  // + byte offset >> 4 selects buffer / half / k-step
      const uint64_t nd0 = sdesc(Nus, 128, 256);
      int kg = 0, it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        mbar_wait_spin(band_full + (it & 1), (it >> 1) & 1);
        const int nc = (tinfo[it & 1].nwalk + R - 1) / R;
        auto mma1 = [&](int kk) {  // D1[kk&1] = NvA . X(kk)   (3xTF32)
          mbar_wait_spin(xfull + (kk & 1), (kk >> 1) & 1);
          if (TM::D1B == 1 && kk >= 1) mbar_wait_spin(d1free + ((kk - 1) & 1), ((kk - 1) >> 1) & 1);
          fence_after_sync();
          const uint32_t d = tbase + TM::D1 + 32 * (kk % TM::D1B);
          const uint64_t xh = xd0 + (uint64_t)(((kk & 1) * (2 * 32 * KJ * 4)) >> 4);
          const uint64_t xl = xh + (uint64_t)((32 * KJ * 4) >> 4);
#pragma unroll
          for (int st = 0; st < KJ / 8; ++st) mma_tf32_ts(d, tbase + TM::NvHi + 8 * st, xh + 16 * st, id1, st > 0);
#pragma unroll
          for (int st = 0; st < KJ / 8; ++st) mma_tf32_ts(d, tbase + TM::NvHi + 8 * st, xl + 16 * st, id1, 1u);
#pragma unroll
          for (int st = 0; st < KJ / 8; ++st) mma_tf32_ts(d, tbase + TM::NvLo + 8 * st, xh + 16 * st, id1, 1u);
          commit(d1full + (kk & 1));
        };
        auto mma2 = [&](int kk, bool first) {  // D2_c += G_c(kk) . Nu(kk)   (3xTF32), c = x, y, z, w
          mbar_wait_spin(gfull + (kk & 1), (kk >> 1) & 1);
          fence_after_sync();
          const uint64_t nh = nd0 + (uint64_t)(((kk % 3) * (2 * NI * R * 4)) >> 4);
          const uint64_t nl = nh + (uint64_t)((NI * R * 4) >> 4);
#pragma unroll
          const uint32_t ga = tbase + TM::G + 64 * (kk % TM::GB);
          for (int c = 0; c < 4; ++c) {
            const uint32_t d = tbase + TM::D2 + NI * c;
            mma_tf32_ts(d, ga + 8 * c, nh, id2, first ? 0u : 1u);
            mma_tf32_ts(d, ga + 8 * c, nl, id2, 1u);
            mma_tf32_ts(d, ga + 32 + 8 * c, nh, id2, 1u);
          }
          commit(m2done + (kk & 1));
        };
        if (nc > 0) {
          mma1(kg);
          for (int k = 0; k < nc; ++k) {
            if (k + 1 < nc) mma1(kg + k + 1);
            mma2(kg + k, k == 0);
          }
        }
        kg += nc;
        mbar_arrive(band_empty + (it & 1));  // every MMA of the tile is issued
      }
    }
  } else {
    // ================================ compute warps: thread / TMEM lane = sample column b
    const uint32_t lane_base = tbase + ((uint32_t)(32 * warp) << 16);
    // per-thread constant smem offsets of the B operands (K-major core-matrix layout)
    const int ap = tid >> 4;          // chunk row written by this thread (X, Nu)
    const int jq = tid & 15;          // band column (X) / band row (Nu) written by this thread
    uint32_t xoff[KJ / 16][4];
#pragma unroll
    for (int h = 0; h < KJ / 16; ++h)
#pragma unroll
      for (int c = 0; c < 4; ++c) xoff[h][c] = kmaj_off(ap * 4 + c, jq + 16 * h, KJ);
    const uint32_t nuoff = kmaj_off(jq, ap, R);
    const int io_off = IO == 2 ? (tid >> 6) * (R * kHRow) + (tid & 63) * 3 : tid * 3;
    constexpr int io_stride = IO == 2 ? kHRow : kSRow;

    int kg = 0, it = 0, last_cb = -1;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int buf = it & 1;
      mbar_wait_spin(band_full + buf, (it >> 1) & 1);
      const TileInfo ti = tinfo[buf];
      const int s = ti.s, rb = ti.rb, cb = ti.cb;
      const int B0 = cb * kCB, cols = min(kCB, C.ns - B0);
      const int S0 = P + rb * prm.K, S1 = min(S0 + prm.K, Rr.n);
      const int band_lo = S0 - P, band_rows = S1 - band_lo;
      const int a_lo = ti.a_lo, nwalk = ti.nwalk, jlo = ti.jlo, ncol = ti.ncol;
      const int nc = (nwalk + R - 1) / R;
      const float* Uk = Rr.knots + (long long)s * Rr.kstride;
      const float4* band = band0 + buf * (NI * KJ);
      const bool valid = tid < cols;

      // ---- column spans, bases and NvA (TMEM A operand of MMA1): only when the column block
      // or the knots change (config 4: once per CTA). The previous tile's MMAs are complete
      // (its last m2done was waited) and its B2 gather is finished (barrier below).
      bar_compute();
      if (it == 0 || cb != last_cb || C.kstride != 0) {
        const float* Vk = C.tspan ? nullptr : C.knots + (long long)s * C.kstride;
        const int b = B0 + (valid ? tid : cols - 1);
        int sv;
        float nv[Q + 1];
        if (C.tspan) {
          sv = __ldg(C.tspan + b);
          const float* tn = C.tN + (size_t)b * C.tnp;
#pragma unroll
          for (int h = 0; h <= Q; ++h) nv[h] = __ldg(tn + h);
        } else {
          const float vb = __ldg(C.s + b);
          sv = d_find_span(Vk, m, Q, vb);
          d_basis<Q>(Vk, sv, vb, Q, nv);
        }
        sv = min(max(sv, Q), m - 1);
        sv = min(max(sv, jlo + Q), jlo + ncol - 1);  // memory safety for unsorted v (R: header)
        sv_s[tid] = sv;
#pragma unroll
        for (int h = 0; h < NQ; ++h) Nv_s[tid * NQ + h] = h <= Q ? nv[h <= Q ? h : 0] : 0.f;
        // NvA row: Nv[b][jlo + jj] for jj < KJ, split hi / lo (KJ = 16: one 32-column store)
        float vh[32], vl[32];
        const int j0 = sv - Q - jlo;
#pragma unroll
        for (int jj = 0; jj < 32; ++jj) {
          float x = 0.f;
#pragma unroll
          for (int h = 0; h <= Q; ++h) x = (jj == j0 + h) ? nv[h] : x;
          x = valid ? x : 0.f;
          vh[jj] = tf32_hi(x);
          vl[jj] = x - vh[jj];
        }
        if constexpr (KJ == 16) {
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) vh[16 + jj] = vl[jj];
          st32(lane_base + TM::NvHi, vh);
        } else {
          st32(lane_base + TM::NvHi, vh);
          st32(lane_base + TM::NvLo, vl);
        }
        last_cb = cb;
      }

      // the band in homogeneous form for the X products (ordered before X(0) by the
      // row-table barriers in write_x)
      for (int x = tid; x < band_rows * KJ; x += kCB) {
        const int ii = x / KJ, jj = x - ii * KJ;
        if (jj < ncol) bandh[ii * KJ + jj] = homog(band[(size_t)ii * CBW + jj]);
      }

      // row span / basis tables of the tile's rows, in windows of kRowChunk rows
      auto stage_rows = [&](int r0) {
        const int cn = min(kRowChunk, nwalk - r0);
        if (tid < cn) {
          const int a = a_lo + r0 + tid;
          int su;
          float nu[P + 1];
          if (Rr.tspan) {
            su = __ldg(Rr.tspan + a);
            const float* tn = Rr.tN + (size_t)a * Rr.tnp;
#pragma unroll
            for (int k = 0; k <= P; ++k) nu[k] = __ldg(tn + k);
          } else {
            const float ua = __ldg(Rr.s + a);
            su = d_find_span(Uk, Rr.n, P, ua);
            d_basis<P>(Uk, su, ua, P, nu);
          }
          su_s[tid] = min(max(su, S0), S1 - 1);  // memory safety for inconsistent inputs
          *reinterpret_cast<float4*>(Nu_s + tid * 4) =
              make_float4(nu[0], P >= 1 ? nu[P >= 1 ? 1 : 0] : 0.f, P >= 2 ? nu[P >= 2 ? 2 : 0] : 0.f,
                          P >= 3 ? nu[P >= 3 ? 3 : 0] : 0.f);
        }
      };
      // X(k) and Nu(k) into smem (B operands of MMA1 / MMA2), split hi / lo; kk = global chunk
      auto write_x = [&](int k, int kk) {
        const int r0 = k * R;
        if (r0 % kRowChunk == 0) {
          bar_compute();  // the previous window is no longer read
          stage_rows(r0);
          bar_compute();
        }
        const int ci = r0 % kRowChunk + ap;
        const bool rv = r0 + ap < nwalk;
        int su = S0;
        float4 n4 = f4(0.f);
        if (rv) {
          su = su_s[ci];
          n4 = *reinterpret_cast<const float4*>(Nu_s + ci * 4);
        }
        const float nu[4] = {n4.x, n4.y, n4.z, n4.w};
        unsigned char* xh = Xs + (kk & 1) * (2 * 32 * KJ * 4);
        unsigned char* xl = xh + 32 * KJ * 4;
        const float4* brow = bandh + (size_t)(su - P - band_lo) * KJ;
#pragma unroll
        for (int h = 0; h < KJ / 16; ++h) {
          const int jj = jq + 16 * h;
          float4 x = f4(0.f);
          if (rv && jj < ncol) {
#pragma unroll
            for (int r = 0; r <= P; ++r) x = fma4v(nu[r], brow[r * KJ + jj], x);
          }
          const float h0 = tf32_hi(x.x), h1 = tf32_hi(x.y), h2 = tf32_hi(x.z), h3 = tf32_hi(x.w);
          *reinterpret_cast<float*>(xh + xoff[h][0]) = h0;
          *reinterpret_cast<float*>(xh + xoff[h][1]) = h1;
          *reinterpret_cast<float*>(xh + xoff[h][2]) = h2;
          *reinterpret_cast<float*>(xh + xoff[h][3]) = h3;
          *reinterpret_cast<float*>(xl + xoff[h][0]) = x.x - h0;
          *reinterpret_cast<float*>(xl + xoff[h][1]) = x.y - h1;
          *reinterpret_cast<float*>(xl + xoff[h][2]) = x.z - h2;
          *reinterpret_cast<float*>(xl + xoff[h][3]) = x.w - h3;
        }
        {  // Nu(k): [16 control rows][8 chunk rows], dense over the band
          unsigned char* nh = Nus + (kk % 3) * (2 * NI * R * 4);
          const int r = band_lo + jq - (su - P);
          float v = 0.f;
#pragma unroll
          for (int rr = 0; rr <= P; ++rr) v = (rv && r == rr) ? nu[rr] : v;
          const float hi = tf32_hi(v);
          *reinterpret_cast<float*>(nh + nuoff) = hi;
          *reinterpret_cast<float*>(nh + NI * R * 4 + nuoff) = v - hi;
        }
        fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor cores
        if (k == 0) {         // NvA TMEM stores (if any) complete before MMA1 of the tile
          wait_st();
          fence_before_sync();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(xfull + (kk & 1));
      };

      const float* gdirect = prm.gout + (((size_t)s * Rr.ns + a_lo) * C.ns + B0 + (valid ? tid : 0)) * 3;
      if (nc > 0) write_x(0, kg);
      for (int k = 0; k < nc; ++k) {
        const int kk = kg + k;
        if (k + 1 < nc) write_x(k + 1, kk + 1);
        mbar_wait_spin(d1full + (kk & 1), (kk >> 1) & 1);
        fence_after_sync();
        float sp[32];
        ld32(lane_base + TM::D1 + 32 * (kk % TM::D1B), sp);
        wait_ld();
        if constexpr (TM::D1B == 1) {  // D1 may be overwritten by MMA1(kk + 1)
          fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(d1free + (kk & 1));
        }
        const int slot = kk % NSTG;
        const float* io = stage + slot * (R * kSRow) + io_off;
        if constexpr (IO >= 1) mbar_wait_spin(sfull + slot, (kk / NSTG) & 1);
        float gh[32], gl[32];
        const bool full = valid && (k * R + R <= nwalk);
        // G = (g/W, -(g.S)/W), S = S'_xyz / W (Eq.8/9 through the homogeneous point), split
        auto row = [&](int r, bool ok) {
          float gx = 0.f, gy = 0.f, gz = 0.f;
          if constexpr (IO >= 1) {
            gx = io[r * io_stride + 0];
            gy = io[r * io_stride + 1];
            gz = io[r * io_stride + 2];
          } else if (ok) {
            const float* gp = gdirect + (size_t)(k * R + r) * C.ns * 3;
            gx = __ldg(gp + 0);
            gy = __ldg(gp + 1);
            gz = __ldg(gp + 2);
          }
          const float Sx = sp[r * 4 + 0], Sy = sp[r * 4 + 1], Sz = sp[r * 4 + 2], W = sp[r * 4 + 3];
          float rw = rcp_approx(W);
          if (!ok) {  // columns past the block / rows past the tile: G = 0 (stale smem, W = 0)
            rw = 0.f;
            gx = gy = gz = 0.f;
          }
          const float G0 = gx * rw, G1 = gy * rw, G2 = gz * rw;
          const float gS = fmaf(G0, Sx, fmaf(G1, Sy, G2 * Sz));
          const float G3 = -gS * rw;
          gh[0 * R + r] = tf32_hi(G0);
          gh[1 * R + r] = tf32_hi(G1);
          gh[2 * R + r] = tf32_hi(G2);
          gh[3 * R + r] = tf32_hi(G3);
          gl[0 * R + r] = G0 - gh[0 * R + r];
          gl[1 * R + r] = G1 - gh[1 * R + r];
          gl[2 * R + r] = G2 - gh[2 * R + r];
          gl[3 * R + r] = G3 - gh[3 * R + r];
        };
        if (full) {
#pragma unroll
          for (int r = 0; r < R; ++r) row(r, true);
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) row(r, valid && (k * R + r < nwalk));
        }
        if (kk >= TM::GB) {  // MMA2(kk - GB) has read this G buffer
          const int kp = kk - TM::GB;
          mbar_wait_spin(m2done + (kp & 1), (kp >> 1) & 1);
          fence_after_sync();
        }
        st32(lane_base + TM::G + 64 * (kk % TM::GB), gh);
        st32(lane_base + TM::G + 64 * (kk % TM::GB) + 32, gl);
        wait_st();
        fence_before_sync();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(gfull + (kk & 1));
          if constexpr (IO >= 1) mbar_arrive(sempty + slot);
        }
      }

      // ---- H = D2 (TMEM) -> smem [b][i]
      float hv[64];
      if (nc > 0) {
        mbar_wait_spin(m2done + ((kg + nc - 1) & 1), ((kg + nc - 1) >> 1) & 1);
        fence_after_sync();
        float h0[32], h1[32];
        ld32(lane_base + TM::D2, h0);
        ld32(lane_base + TM::D2 + 32, h1);
        wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          hv[i] = h0[i];
          hv[32 + i] = h1[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i) hv[i] = 0.f;
      }
      kg += nc;
      if (tid < KJ) {  // samples b whose basis touches control column j = jlo + tid
        const int j = jlo + tid;
        int lo2 = 0, hi2 = cols;
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2) >> 1;
          if (sv_s[mid] < j) lo2 = mid + 1; else hi2 = mid;
        }
        int e2 = lo2, eh = cols;
        while (e2 < eh) {
          const int mid = (e2 + eh) >> 1;
          if (sv_s[mid] <= j + Q) e2 = mid + 1; else eh = mid;
        }
        jb[tid] = make_int2(lo2, e2);
      }

      // ---- B2: dQ[i][j] = sum_b Nv[b][j - sv(b) + q] H[b][i], ascending b; then the epilogue.
      // H goes through smem in two halves of NH control rows.
      float4* gctrl_s = prm.gctrl + (size_t)s * Rr.n * m;
      float4* slots = prm.slots ? prm.slots + (((size_t)s * prm.NRB + rb) * prm.NCB + cb) * prm.T_rows * m : nullptr;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        bar_compute();  // jb ready / the previous half's gather done
#pragma unroll
        for (int ii = 0; ii < NH; ++ii) {
          const int i2 = half * NH + ii;
          Hs[tid * NH + ii] = make_float4(hv[i2], hv[NI + i2], hv[2 * NI + i2], hv[3 * NI + i2]);
        }
        bar_compute();
        for (int o = tid; o < NH * KJ; o += kCB) {
          const int ih = o & (NH - 1), jj = o / NH;
          const int ii = half * NH + ih;
          if (ii >= band_rows || jj >= ncol) continue;
          const int j = jlo + jj;
          const int2 r2 = jb[jj];
          float4 a4 = f4(0.f);
          for (int bb = r2.x; bb < r2.y; ++bb) {
            const int h = j - sv_s[bb] + Q;  // in [0, Q] for sorted v; guarded for unsorted v
            if (h >= 0 && h <= Q) a4 = fma4v(Nv_s[bb * NQ + h], Hs[bb * NH + ih], a4);
          }
          const int i = band_lo + ii;
          if (prm.direct) {  // dP = w dQ_xyz, dw = P.dQ_xyz + dQ_w
            const float4 c = band[(size_t)ii * CBW + jj];
            gctrl_s[(size_t)i * m + j] =
                make_float4(c.w * a4.x, c.w * a4.y, c.w * a4.z, fmaf(c.x, a4.x, fmaf(c.y, a4.y, fmaf(c.z, a4.z, a4.w))));
          } else {
            slots[(size_t)ii * m + j] = a4;
          }
        }
      }
      if (prm.direct) {  // control columns this block does not touch (every row is in the band)
        for (int x = tid; x < band_rows * m; x += kCB) {
          const int ii = x / m, j = x - ii * m;
          if (j < jlo || j >= jlo + ncol) gctrl_s[(size_t)(band_lo + ii) * m + j] = f4(0.f);
        }
        if (prm.gR && s < prm.gR_items)  // knot gradients are zero by definition
          for (int x = tid; x < prm.gR_per; x += kCB) prm.gR[(size_t)s * prm.gR_per + x] = 0.f;
        if (prm.gC && s < prm.gC_items)
          for (int x = tid; x < prm.gC_per; x += kCB) prm.gC[(size_t)s * prm.gC_per + x] = 0.f;
      } else if (rb == 0 && tid == 0) {
        prm.colband[(size_t)s * prm.NCB + cb] = make_int2(jlo, jlo + ncol - 1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(band_empty + buf);  // this warp is done with the band
    }
  }

  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (warp == 0) tmem_dealloc(tbase, kTmemCols);
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      n = v;
    else
      n = 148;
  }
  return n;
}

template <int P, int Q, int KJ, int IO>
static cudaError_t launch_k(const Params& prm, cudaStream_t st) {
  constexpr int NQ = (Q + 1) <= 4 ? 4 : 8;
  const size_t smem = Layout<KJ, NQ>::bytes;
  static bool attr_set[64] = {};
  int dev = 0;
  cudaError_t e0 = cudaGetDevice(&dev);
  if (e0 != cudaSuccess) return e0;
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(nurbs_bwd_tc_kernel<P, Q, KJ, IO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  const long long ntiles = (long long)prm.B * prm.NRB * prm.NCB;
  if (ntiles > 0x7fffffffLL) return cudaErrorInvalidValue;
  const long long grid = ntiles < 2LL * num_sms() ? ntiles : 2LL * num_sms();
  nurbs_bwd_tc_kernel<P, Q, KJ, IO><<<(unsigned)grid, kThr, smem, st>>>(prm, (int)ntiles);
  return cudaGetLastError();
}

template <int P, int Q, int KJ>
static cudaError_t launch_kj(const Params& prm, cudaStream_t st) {
  if (prm.bulk && prm.tmap) return launch_k<P, Q, KJ, 2>(prm, st);
  if (prm.bulk) return launch_k<P, Q, KJ, 1>(prm, st);
  return launch_k<P, Q, KJ, 0>(prm, st);
}

}  // namespace tc

// The tensor-core backward covers bicubic surfaces whose control net has at most 32 columns
// (every 128-sample column block's band then fits the MMA's K) and bands of <= 16 rows (the
// plan guarantees it); other shapes return cudaErrorNotSupported and run the SIMT kernel.
bool bwd_tc_supported(const Params& prm, int P, int q) {
  return P == 3 && q == 3 && prm.c.n <= 32 && prm.T_rows <= tc::NI && prm.CBW == prm.c.n;
}

cudaError_t launch_bwd_tc(const Params& prm, int P, int q, cudaStream_t st) {
  if (!bwd_tc_supported(prm, P, q)) return cudaErrorNotSupported;
  if (prm.c.n <= 16) return tc::launch_kj<3, 3, 16>(prm, st);
  return tc::launch_kj<3, 3, 32>(prm, st);
}

}  // namespace nb
