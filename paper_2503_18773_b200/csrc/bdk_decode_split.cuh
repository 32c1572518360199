// bdk_decode_split.cuh -- fast decode with split consumers (included by
// bdk_decode_fast.cu inside its anonymous namespace; reuses its helpers).
//
// Same schedule, ring, prep warp, partial slots, merge and fused flush as
// decode_fast_kernel, but each 16-byte chunk j of the block rows is served by
// a PAIR of warps instead of one:
//   QK warp j  S^T = codes_K . Q'^T, online softmax (the pair's running max,
//              sums and zero term), P' = P s_t 2^(2-sh) as P'^T B-fragments,
//              handed over in a shared-memory slot with the O rescale factors;
//   PV warp j  O^T += codes_V^T . P'^T (the pair's O accumulator), then the
//              segment's finalize / completion count / merge / flush.
// The work per pair equals one warp's of the fused kernel (same extraction,
// same MMAs, same numerics, bit-identical results), but each warp keeps half
// the live state (no O accumulator in QK warps, no Q' fragments in PV
// warps), so a CTA runs 2 W_n consumer warps at <= 96 registers and the SM
// twice as many consumer warps to hide the extraction -> MMA latencies that
// bound the 2-bit kernel.  Residual tiles (fp16 window) flow
// through the same pair pipeline.

// P hand-over slot: P'^T B-fragments [2 * NPAIR <= 8][32 lanes] u32, O rescale
// factors [2][32] f32, "max moved" flag
constexpr int PS_WORDS = 8 * 32 + 2 * 32 + 4;

struct SplitSmem {
  uint32_t ring, prep, merge, pslot, stslot, bars, total;
  uint32_t prep_stride, merge_floats;
};

__host__ __device__ inline SplitSmem split_layout(const Geom& G, int ng, int NS, int WN) {
  SplitSmem L;
  const int gpb = G.n_r / G.g;
  L.ring = 0;
  L.prep_stride = (uint32_t)((gpb * QP_BYTES + 127) / 128 * 128);
  L.prep = L.ring + NS * G.rec_bytes;
  L.merge = L.prep + NS * L.prep_stride;
  const uint32_t merge_bytes =
      (uint32_t)(max(WN * (ng * D + 16), 24 + 2 * MERGE_KC * 8 + 4 * 32 * WN) * 4 + 64);
  L.merge_floats = merge_bytes / 4;
  L.pslot = L.merge + merge_bytes;                                    // [WN][2]
  L.stslot = L.pslot + (uint32_t)(WN * 2 * PS_WORDS * 4);             // [WN][6][32] f32
  L.bars = (L.stslot + (uint32_t)(WN * 6 * 32 * 4) + 7) / 8 * 8;
  // full, empty, ready [NS]; pfull, pempty [WN][2]; stfull, stempty [WN]; flag
  L.total = L.bars + (uint32_t)((3 * NS + 6 * WN) * 8 + 16);
  return L;
}

// online softmax for a QK warp: like softmax_update, but the O rescale is
// returned (r0, r1) for the PV warp instead of applied; true if the max moved
template <int NPAIR>
__device__ __forceinline__ bool softmax_split(float (&x)[NPAIR][4], Soft& st, float& r0,
                                              float& r1) {
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int i = 0; i < NPAIR; ++i) {
    mx0 = fmaxf(mx0, fmaxf(x[i][0], x[i][2]));
    mx1 = fmaxf(mx1, fmaxf(x[i][1], x[i][3]));
  }
  bool moved = false;
  r0 = r1 = 1.f;
  if (__any_sync(0xffffffffu, mx0 > st.m0 + TAU || mx1 > st.m1 + TAU)) {
#pragma unroll
    for (int off = 4; off <= 16; off <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
    }
    const float mn0 = fmaxf(st.m0, mx0), mn1 = fmaxf(st.m1, mx1);
    r0 = st.m0 == -INFINITY ? 0.f : ex2(st.m0 - mn0);
    r1 = st.m1 == -INFINITY ? 0.f : ex2(st.m1 - mn1);
    st.l0 *= r0;
    st.l1 *= r1;
    st.z0 *= r0;
    st.z1 *= r1;
    st.m0 = mn0;
    st.m1 = mn1;
    moved = true;
  }
  const float b0 = st.m0 == -INFINITY ? 0.f : st.m0;
  const float b1 = st.m1 == -INFINITY ? 0.f : st.m1;
#pragma unroll
  for (int i = 0; i < NPAIR; ++i) {
    x[i][0] = ex2(x[i][0] - b0);
    x[i][1] = ex2(x[i][1] - b1);
    x[i][2] = ex2(x[i][2] - b0);
    x[i][3] = ex2(x[i][3] - b1);
    st.l0 += x[i][0] + x[i][2];
    st.l1 += x[i][1] + x[i][3];
  }
  return moved;
}

__device__ __forceinline__ void ps_put_rescale(uint32_t* ps, bool moved, float r0, float r1) {
  const int lane = threadIdx.x & 31;
  float* pf = reinterpret_cast<float*>(ps);
  pf[8 * 32 + lane] = r0;
  pf[9 * 32 + lane] = r1;
  if (lane == 0) ps[10 * 32] = moved ? 1u : 0u;
}

// PV side: apply a pending O rescale of the slot
__device__ __forceinline__ void ps_rescale_o(const uint32_t* ps, float (&o)[OT][4]) {
  if (ps[10 * 32]) {  // warp-uniform
    const int lane = threadIdx.x & 31;
    const float* pf = reinterpret_cast<const float*>(ps);
    const float r0 = pf[8 * 32 + lane], r1 = pf[9 * 32 + lane];
#pragma unroll
    for (int mt = 0; mt < OT; ++mt) {
      o[mt][0] *= r0;
      o[mt][1] *= r1;
      o[mt][2] *= r0;
      o[mt][3] *= r1;
    }
  }
}

// QK warp, one packed block (chunk j): S^T, softmax, P' -> slot ps.  Frees
// the stage's K words, V params and prep slot (empty_s).
template <int BITS, int WN>
__device__ __forceinline__ void qk_block(const uint8_t* rec, const uint8_t* qp, const Geom& G, int j,
                                         float scale, const int (&vtok)[(16 / BITS) / 2][2],
                                         Soft& st, uint32_t* ps, uint64_t* empty_s) {
  constexpr int P = 16 / BITS, NPAIR = P / 2, RB = 16 * WN;
  constexpr int SH_REF = BITS == 8 ? 0 : 2;
  const int lane = threadIdx.x & 31, gid = lane >> 2, t4 = lane & 3;
  const uint32_t* vpr = reinterpret_cast<const uint32_t*>(rec + 2 * G.wbytes + G.kp_bytes);
  uint32_t qb[KT][2];
  {
    const int mi = lane >> 3, r = lane & 7;
#pragma unroll
    for (int kk = 0; kk < KT / 2; ++kk) {
      const int kt = 2 * kk + (mi >> 1);
      const int cof = (kt * 16 + (mi & 1) * 8) * 2;
      ldsm_x4(smem_u32(qp + r * QP_ROW + cof), qb[2 * kk][0], qb[2 * kk][1], qb[2 * kk + 1][0],
              qb[2 * kk + 1][1]);
    }
  }
  const float2 zz = *reinterpret_cast<const float2*>(qp + 8 * QP_ROW + 8 * t4);
  const float zs0 = zz.x * scale, zs1 = zz.y * scale;
  constexpr bool KSPLIT = NPAIR <= 2;
  constexpr int NCH = NPAIR * (KSPLIT ? 2 : 1);
  float chn[NCH][4];
#pragma unroll
  for (int i = 0; i < NCH; ++i) chn[i][0] = chn[i][1] = chn[i][2] = chn[i][3] = 0.f;
  {
    const uint32_t kw = smem_u32(rec);
    uint32_t kr[4][4];
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      const int row = kc * 32 + lane;
      ldsm_x4_t(kw + row * RB + ((j ^ swz(row, WN)) << 4), kr[kc][0], kr[kc][1], kr[kc][2],
                kr[kc][3]);
    }
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const uint32_t rl = kr[kt / 2][2 * (kt % 2)], rh = kr[kt / 2][2 * (kt % 2) + 1];
      const uint32_t rl8 = rl >> 8, rh8 = rh >> 8;
#pragma unroll
      for (int pi = 0; pi < NPAIR; ++pi) {
        uint32_t af[4];
#define BDK_KEXT(PI)                                 \
  if (pi == PI) {                                    \
    af[0] = ext_sub<BITS, (2 * PI) % P>(rl, rl8);     \
    af[1] = ext_sub<BITS, (2 * PI + 1) % P>(rl, rl8); \
    af[2] = ext_sub<BITS, (2 * PI) % P>(rh, rh8);     \
    af[3] = ext_sub<BITS, (2 * PI + 1) % P>(rh, rh8); \
  }
        BDK_KEXT(0)
        BDK_KEXT(1)
        BDK_KEXT(2)
        BDK_KEXT(3)
#undef BDK_KEXT
        mma16816(chn[pi + NPAIR * (KSPLIT ? (kt & 1) : 0)], af, qb[kt][0], qb[kt][1]);
      }
    }
  }
  float sacc[NPAIR][4];
#pragma unroll
  for (int i = 0; i < NPAIR; ++i)
#pragma unroll
    for (int r = 0; r < 4; ++r) sacc[i][r] = KSPLIT ? chn[i][r] + chn[i + NPAIR][r] : chn[i][r];
#pragma unroll
  for (int i = 0; i < NPAIR; ++i) {
    const float al = scale * (float)(1 << (24 - ((2 * i) % P) * BITS % 8));
    const float ah = scale * (float)(1 << (24 - ((2 * i + 1) % P) * BITS % 8));
    sacc[i][0] = fmaf(sacc[i][0], al, zs0);
    sacc[i][1] = fmaf(sacc[i][1], al, zs1);
    sacc[i][2] = fmaf(sacc[i][2], ah, zs0);
    sacc[i][3] = fmaf(sacc[i][3], ah, zs1);
  }
  float r0, r1;
  const bool moved = softmax_split<NPAIR>(sacc, st, r0, r1);
#pragma unroll
  for (int i = 0; i < NPAIR; ++i) {
    const int g0 = (8 * j + gid) * P;
    const float2 pa = __half22float2(u2h(vpr[g0 + vtok[i][0]]));
    const float2 pz = __half22float2(u2h(vpr[g0 + vtok[i][1]]));
    const float sz0 = pa.x * (float)(1 << (SH_REF + 8)) / (float)(1 << (8 + ((2 * i) % P) * BITS % 8));
    const float sz1 =
        pz.x * (float)(1 << (SH_REF + 8)) / (float)(1 << (8 + ((2 * i + 1) % P) * BITS % 8));
    st.z0 = fmaf(sacc[i][0], pa.y, fmaf(sacc[i][2], pz.y, st.z0));
    st.z1 = fmaf(sacc[i][1], pa.y, fmaf(sacc[i][3], pz.y, st.z1));
    ps[(2 * i) * 32 + lane] = movmatrix_t(pack_h2(sacc[i][0] * sz0, sacc[i][1] * sz0));
    ps[(2 * i + 1) * 32 + lane] = movmatrix_t(pack_h2(sacc[i][2] * sz1, sacc[i][3] * sz1));
  }
  ps_put_rescale(ps, moved, r0, r1);
  __syncwarp();
  if (lane == 0) mbar_arrive(empty_s);
}

// PV warp, one packed block (chunk j): O^T += codes_V^T . P'^T.  Frees the
// stage's V words (empty_s) and the P slot (pempty_b).
template <int BITS, int WN>
__device__ __forceinline__ void pv_block(const uint8_t* vwords, int j, const uint32_t* ps,
                                         float (&o)[OT][4], uint64_t* empty_s, uint64_t* pempty_b) {
  constexpr int P = 16 / BITS, NPAIR = P / 2, RB = 16 * WN;
  const int lane = threadIdx.x & 31;
  uint32_t vr[4][4];
  const uint32_t vw = smem_u32(vwords);
#pragma unroll
  for (int vc = 0; vc < 4; ++vc) {
    const int row = vc * 32 + lane;
    ldsm_x4(vw + row * RB + ((j ^ swz(row, WN)) << 4), vr[vc][0], vr[vc][1], vr[vc][2], vr[vc][3]);
  }
  uint32_t pb[NPAIR][2];
#pragma unroll
  for (int i = 0; i < NPAIR; ++i) {
    pb[i][0] = ps[(2 * i) * 32 + lane];
    pb[i][1] = ps[(2 * i + 1) * 32 + lane];
  }
  ps_rescale_o(ps, o);
  __syncwarp();
  if (lane == 0) {
    mbar_arrive(empty_s);
    mbar_arrive(pempty_b);
  }
#pragma unroll
  for (int mt = 0; mt < KT; ++mt) {
    const uint32_t ra = vr[mt / 2][2 * (mt % 2)], rb = vr[mt / 2][2 * (mt % 2) + 1];
    const uint32_t ra8 = ra >> 8, rb8 = rb >> 8;
#pragma unroll
    for (int pi = 0; pi < NPAIR; ++pi) {
      uint32_t af[4];
#define BDK_VEXT(PI)                                 \
  if (pi == PI) {                                    \
    af[0] = ext_sub<BITS, (2 * PI) % P>(ra, ra8);     \
    af[1] = ext_sub<BITS, (2 * PI) % P>(rb, rb8);     \
    af[2] = ext_sub<BITS, (2 * PI + 1) % P>(ra, ra8); \
    af[3] = ext_sub<BITS, (2 * PI + 1) % P>(rb, rb8); \
  }
      BDK_VEXT(0)
      BDK_VEXT(1)
      BDK_VEXT(2)
      BDK_VEXT(3)
#undef BDK_VEXT
      mma16816(o[mt], af, pb[pi][0], pb[pi][1]);
    }
  }
}

template <int BITS, int WN, int NS>
__global__ void __maxnreg__(96) decode_split_kernel(const __grid_constant__ DevCache c,
                                                    const __grid_constant__ FastArgs a) {
  constexpr int P = 16 / BITS, NPAIR = P / 2;
  constexpr int NCON = 2 * WN;  // PV warps [0, WN), QK warps [WN, 2 WN)
  constexpr int RT = 16 * WN;   // residual tokens per unit (a 16-token tile per pair)
  constexpr int SH_REF = BITS == 8 ? 0 : 2;
  const float oscale = exp2f((float)(24 - SH_REF));
  extern __shared__ __align__(1024) uint8_t smem[];
  const Geom& G = c.G;
  const int cells = G.batch * G.heads_kv;
  const int ng = a.n_group;
  const SplitSmem L = split_layout(G, ng, NS, WN);
  uint8_t* ring = smem + L.ring;
  uint8_t* prep = smem + L.prep;
  float* merge_sm = reinterpret_cast<float*>(smem + L.merge);
  uint32_t* pslot = reinterpret_cast<uint32_t*>(smem + L.pslot);
  float* stslot = reinterpret_cast<float*>(smem + L.stslot);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + NS;
  uint64_t* ready = empty + NS;
  uint64_t* pfull = ready + NS;        // [WN][2]
  uint64_t* pempty = pfull + 2 * WN;   // [WN][2]
  uint64_t* stfull = pempty + 2 * WN;  // [WN]
  uint64_t* stempty = stfull + WN;     // [WN]
  int* flag = reinterpret_cast<int*>(stempty + WN);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, t4 = lane & 3;
  const int REC = G.rec_bytes;

  for (uint32_t i = threadIdx.x * 16; i < NS * L.prep_stride; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(prep + i) = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2 * WN);  // the QK and the PV warp of every chunk
      mbar_init(&ready[s], 1);
    }
    for (int i = 0; i < 2 * WN; ++i) {
      mbar_init(&pfull[i], 1);
      mbar_init(&pempty[i], 1);
    }
    for (int i = 0; i < WN; ++i) {
      mbar_init(&stfull[i], 1);
      mbar_init(&stempty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  pdl_launch_dependents();

  const Sched S = make_sched(c, a, cells, RT);
  SchedOut so;
  if (a.dev_sched) {
    if (a.pdl) pdl_wait();
    so = sched_scan(S, cells, reinterpret_cast<long long*>(merge_sm));
  } else {
    so = sched_host(S, a, cells);
  }
  const long long T = so.T;
  const int N = (int)min((long long)gridDim.x, T);
  const long long u_begin = (int)blockIdx.x < N ? (long long)blockIdx.x * T / N : T;
  const long long u_end = (int)blockIdx.x < N ? (long long)(blockIdx.x + 1) * T / N : T;
  const int cell0 = so.cell0;

  // ------------------------------------------------------------ TMA warp
  if (warp == NCON) {
    if (lane == 0 && u_begin < u_end) {
      const uint64_t pol = policy_evict_first();
      bool waited = !a.pdl || a.dev_sched;
      if (!a.prefetch_ok && !waited) {
        pdl_wait();
        waited = true;
      }
      int it = 0;
      long long u = u_begin, off = so.off0;
      for (int cell = cell0; u < u_end; ++cell) {
        const int nbc = S.nb(cell);
        const long long ce = off + S.units(cell, nbc);
        const long long seg_end = min(u_end, ce);
        const long long pk_end = min(seg_end, off + nbc);
        const uint8_t* base = c.records + (size_t)cell * G.max_blocks * REC;
        for (long long x = u; x < pk_end; ++x, ++it) {
          const int s = it % NS;
          if (!waited && it == NS) {
            pdl_wait();
            waited = true;
          }
          if (it >= NS) mbar_wait_sleep(&empty[s], ((it / NS) - 1) & 1);
          mbar_expect_tx(&full[s], (uint32_t)REC);
          const int blk = a.blk_begin + (int)(x - off);
          tma_bulk_g2s(ring + (size_t)s * REC, base + (size_t)blk * REC, (uint32_t)REC, &full[s],
                       pol);
        }
        u = seg_end;
        off = ce;
      }
    }
    return;
  }
  if (a.pdl && !a.dev_sched) pdl_wait();

  // ---------------------------------------------------------- prep warp
  if (warp > NCON) {
    if (u_begin >= u_end) return;
    const int nh = ng <= 1 ? 1 : ng <= 2 ? 2 : ng <= 4 ? 4 : 8;
    PrepCtx px{ring, prep, full, ready, nullptr, REC, (int)L.prep_stride, 0, u_begin, u_end,
               so.off0, cell0, RT};
    if (nh == 1) prep_loop<1, NS, 1>(c, a, px);
    else if (nh == 2) prep_loop<2, NS, 1>(c, a, px);
    else if (nh == 4) prep_loop<4, NS, 1>(c, a, px);
    else prep_loop<8, NS, 1>(c, a, px);
    return;
  }

  const bool qk = warp >= WN;
  const int j = qk ? warp - WN : warp;  // chunk (and residual tile lane) of the pair
  const float scale = a.sm_scale_log2;
  const bool app = a.k_new != nullptr && !a.skip_residual;
  uint64_t* pf_j = pfull + 2 * j;
  uint64_t* pe_j = pempty + 2 * j;
  uint32_t* ps_j = pslot + (size_t)(2 * j) * PS_WORDS;
  float* st_j = stslot + (size_t)j * 6 * 32;

  // ------------------------------------------------------------ QK warps
  if (qk) {
    const int kgr = (8 * j * P) / G.g;
    int vtok[NPAIR][2];
#pragma unroll
    for (int i = 0; i < NPAIR; ++i) {
      vtok[i][0] = pos_token(2 * i, P, G.interleave);
      vtok[i][1] = pos_token(2 * i + 1, P, G.interleave);
    }
    int it = 0, item = 0, seg = 0;
    long long u = u_begin, off = so.off0;
    for (int cell = cell0; u < u_end; ++cell, ++seg) {
      const int nbc = S.nb(cell);
      const long long cb = off, ce = off + S.units(cell, nbc);
      const long long seg_end = min(u_end, ce);
      const long long res_begin = cb + nbc;
      const long long pk_end = min(seg_end, res_begin);
      Soft st{-INFINITY, -INFINITY, 0.f, 0.f, 0.f, 0.f};
      const int it_end = it + (int)max(0LL, pk_end - u);
      for (int k = it; k < it_end; ++k, ++item) {
        const int s = k % NS, b = item & 1;
        mbar_wait(&ready[s], (k / NS) & 1);
        mbar_wait(&full[s], (k / NS) & 1);
        if (item >= 2) mbar_wait(&pe_j[b], ((item >> 1) - 1) & 1);
        qk_block<BITS, WN>(ring + (size_t)s * REC, prep + (size_t)s * L.prep_stride + kgr * QP_BYTES,
                           G, j, scale, vtok, st, ps_j + b * PS_WORDS, &empty[s]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&pf_j[b]);
      }
      it = it_end;
      if (seg_end > res_begin && !a.skip_residual) {
        const int rl0 = a.uni_len ? a.uni_rl : __ldcg(S.rl() + cell);
        const int rlen = rl0 + (app ? 1 : 0);
        const int t_lo = (int)(max(u, res_begin) - res_begin) * RT;
        const int t_hi = min(rlen, (int)(seg_end - res_begin) * RT);
        __half* rk = c.res_k + (size_t)cell * G.n_r * D;
        if (app && rl0 >= t_lo && rl0 < t_hi) {  // append_token: the K row (kvcache.cpp:170-182)
          const __half* kn = a.k_new + (size_t)cell * D;
          for (int i = threadIdx.x - WN * 32; i < D; i += WN * 32) rk[(size_t)rl0 * D + i] = kn[i];
          asm volatile("bar.sync 2, %0;" ::"r"(WN * 32) : "memory");
        }
        const int bidx = cell / G.heads_kv, hk = cell % G.heads_kv;
        uint32_t qb[KT][2];
        {
          const __half* qh = a.q + ((size_t)bidx * a.heads_q + (size_t)hk * ng + gid) * D;
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            qb[kt][0] = gid < ng ? *reinterpret_cast<const uint32_t*>(qh + kt * 16 + 2 * t4) : 0u;
            qb[kt][1] = gid < ng ? *reinterpret_cast<const uint32_t*>(qh + kt * 16 + 8 + 2 * t4) : 0u;
          }
        }
        for (int t0 = t_lo + 16 * j; t0 < t_hi; t0 += RT, ++item) {
          const int b = item & 1;
          if (item >= 2) mbar_wait(&pe_j[b], ((item >> 1) - 1) & 1);
          const bool v0 = t0 + gid < t_hi, v1 = t0 + gid + 8 < t_hi;
          const __half* k0 = rk + (size_t)(t0 + gid) * D + 2 * t4;
          const __half* k1 = k0 + 8 * D;
          float sacc[1][4] = {{0.f, 0.f, 0.f, 0.f}};
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            uint32_t ka[4];
            ka[0] = v0 ? *reinterpret_cast<const uint32_t*>(k0 + kt * 16) : 0u;
            ka[1] = v1 ? *reinterpret_cast<const uint32_t*>(k1 + kt * 16) : 0u;
            ka[2] = v0 ? *reinterpret_cast<const uint32_t*>(k0 + kt * 16 + 8) : 0u;
            ka[3] = v1 ? *reinterpret_cast<const uint32_t*>(k1 + kt * 16 + 8) : 0u;
            mma16816(sacc[0], ka, qb[kt][0], qb[kt][1]);
          }
          sacc[0][0] = v0 ? sacc[0][0] * scale : -INFINITY;
          sacc[0][1] = v0 ? sacc[0][1] * scale : -INFINITY;
          sacc[0][2] = v1 ? sacc[0][2] * scale : -INFINITY;
          sacc[0][3] = v1 ? sacc[0][3] * scale : -INFINITY;
          float r0, r1;
          const bool moved = softmax_split<1>(sacc, st, r0, r1);
          uint32_t* ps = ps_j + b * PS_WORDS;
          ps[0 * 32 + lane] = movmatrix_t(pack_h2(sacc[0][0], sacc[0][1]));
          ps[1 * 32 + lane] = movmatrix_t(pack_h2(sacc[0][2], sacc[0][3]));
          ps_put_rescale(ps, moved, r0, r1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&pf_j[b]);
        }
      }
      // the segment's softmax state -> PV warp j
      if (seg > 0) mbar_wait(&stempty[j], (seg - 1) & 1);
      st_j[0 * 32 + lane] = st.m0;
      st_j[1 * 32 + lane] = st.m1;
      st_j[2 * 32 + lane] = st.l0;
      st_j[3 * 32 + lane] = st.l1;
      st_j[4 * 32 + lane] = st.z0;
      st_j[5 * 32 + lane] = st.z1;
      __syncwarp();
      if (lane == 0) mbar_arrive(&stfull[j]);
      u = seg_end;
      off = ce;
    }
    return;
  }

  // ------------------------------------------------------------ PV warps
  const int stride_slot = slot_stride(ng);
  int it = 0, item = 0, seg = 0;
  long long u = u_begin, off = so.off0;
  for (int cell = cell0; u < u_end; ++cell, ++seg) {
    const int nbc = S.nb(cell);
    const long long cb = off, ce = off + S.units(cell, nbc);
    const long long seg_end = min(u_end, ce);
    const long long res_begin = cb + nbc;
    const long long pk_end = min(seg_end, res_begin);
    float o[OT][4];
#pragma unroll
    for (int mt = 0; mt < OT; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    const int it_end = it + (int)max(0LL, pk_end - u);
    for (int k = it; k < it_end; ++k, ++item) {
      const int s = k % NS, b = item & 1;
      mbar_wait(&full[s], (k / NS) & 1);
      mbar_wait(&pf_j[b], (item >> 1) & 1);
      pv_block<BITS, WN>(ring + (size_t)s * REC + G.wbytes, j, ps_j + b * PS_WORDS, o, &empty[s],
                         &pe_j[b]);
    }
    it = it_end;
    const int rl0 = a.uni_len ? a.uni_rl : __ldcg(S.rl() + cell);
    float oscale_seg = oscale;
    if (seg_end > res_begin && !a.skip_residual) {
#pragma unroll
      for (int mt = 0; mt < KT; ++mt) {
        o[mt][0] *= oscale;
        o[mt][1] *= oscale;
        o[mt][2] *= oscale;
        o[mt][3] *= oscale;
      }
      oscale_seg = 1.f;
      const int rlen = rl0 + (app ? 1 : 0);
      const int t_lo = (int)(max(u, res_begin) - res_begin) * RT;
      const int t_hi = min(rlen, (int)(seg_end - res_begin) * RT);
      __half* rv = c.res_v + (size_t)cell * G.n_r * D;
      if (app && rl0 >= t_lo && rl0 < t_hi) {  // append_token: the V row
        const __half* vn = a.v_new + (size_t)cell * D;
        for (int i = threadIdx.x; i < D; i += WN * 32) rv[(size_t)rl0 * D + i] = vn[i];
        named_bar(1, WN * 32);
      }
      for (int t0 = t_lo + 16 * j; t0 < t_hi; t0 += RT, ++item) {
        const int b = item & 1;
        const bool v0 = t0 + gid < t_hi, v1 = t0 + gid + 8 < t_hi;
        const __half* w0 = rv + (size_t)(t0 + gid) * D + 2 * t4;
        const __half* w1 = w0 + 8 * D;
        mbar_wait(&pf_j[b], (item >> 1) & 1);
        const uint32_t* ps = ps_j + b * PS_WORDS;
        const uint32_t pb0 = ps[0 * 32 + lane], pb1 = ps[1 * 32 + lane];
        ps_rescale_o(ps, o);
        __syncwarp();
        if (lane == 0) mbar_arrive(&pe_j[b]);
#pragma unroll
        for (int mt = 0; mt < KT; ++mt) {
          uint32_t af[4];
          af[0] = movmatrix_t(v0 ? *reinterpret_cast<const uint32_t*>(w0 + mt * 16) : 0u);
          af[1] = movmatrix_t(v0 ? *reinterpret_cast<const uint32_t*>(w0 + mt * 16 + 8) : 0u);
          af[2] = movmatrix_t(v1 ? *reinterpret_cast<const uint32_t*>(w1 + mt * 16) : 0u);
          af[3] = movmatrix_t(v1 ? *reinterpret_cast<const uint32_t*>(w1 + mt * 16 + 8) : 0u);
          mma16816(o[mt], af, pb0, pb1);
        }
      }
    }
    // the pair's softmax state from QK warp j
    mbar_wait(&stfull[j], seg & 1);
    Soft st;
    st.m0 = st_j[0 * 32 + lane];
    st.m1 = st_j[1 * 32 + lane];
    st.l0 = st_j[2 * 32 + lane];
    st.l1 = st_j[3 * 32 + lane];
    st.z0 = st_j[4 * 32 + lane];
    st.z1 = st_j[5 * 32 + lane];
    __syncwarp();
    if (lane == 0) mbar_arrive(&stempty[j]);

    float* slot = a.slots + (size_t)(blockIdx.x + cell) * stride_slot;
    finalize_segment<WN, 1>(st, o, merge_sm, ng, slot, oscale_seg);  // ends with a barrier
    const int lo = cta_of_unit(cb, T, N), hi = cta_of_unit(ce - 1, T, N);
    if (threadIdx.x == 0) {
      const int prev = atom_add_acq_rel_gpu(a.counters + cell, 1);
      const int last = prev == hi - lo;
      if (last) a.counters[cell] = 0;
      flag[0] = !last ? 0 : (app && rl0 + 1 == G.n_r) ? 2 : 1;
    }
    named_bar(1, WN * 32);
    const int commit = flag[0];
    if (commit) {
      const float* base = a.slots + (size_t)(lo + cell) * stride_slot;
      if (hi - lo + 1 <= MERGE_KC_FEW)
        merge_cell_few<WN>(MergeDst{a.out, a.out_lse, a.heads_q, a.n_group}, G, cell, base,
                           hi - lo + 1, merge_sm, nullptr);
      else
        merge_cell<WN, 8>(MergeDst{a.out, a.out_lse, a.heads_q, a.n_group}, G, cell, base,
                          hi - lo + 1, merge_sm, nullptr);
      const int pb0 = a.uni_len ? a.uni_pb : __ldcg(S.pb() + cell);
      if (commit == 2) {
        named_bar(1, WN * 32);
        const size_t wo = (size_t)cell * G.n_r * D;
        uint8_t* rec = c.records + ((size_t)cell * G.max_blocks + pb0) * REC;
        if constexpr ((WN == 2 || WN == 4 || WN == 8) && BITS != 8 && (WN * P) % 16 == 0) {
          qf_flush_window<BITS, WN * 32>(G, c.res_k + wo, c.res_v + wo, rec,
                                         reinterpret_cast<uint8_t*>(merge_sm), 1);
        } else {
          flush_window<BITS>(G, c.res_k + wo, c.res_v + wo, rec, WN * 32, 1);
        }
      }
      if (threadIdx.x == 0) {
        S.pb_n()[cell] = commit == 2 ? pb0 + 1 : pb0;
        S.rl_n()[cell] = commit == 2 ? 0 : rl0 + (app ? 1 : 0);
      }
    }
    named_bar(1, WN * 32);
    u = seg_end;
    off = ce;
  }
}
