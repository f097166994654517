// smo_bincl.cuh -- the SMO solver kernel for exactly binary data resident in one thread-block
// cluster (the latency-bound small-problem path; W2, the bench workload, runs here).
//
// Same method and arithmetic as smo_persistent (readings R13-R16: popcount
// distances are exact, K = ktab[D] = exp_cr(-gamma D), K_ii = ktab[0] = 1), restructured for
// latency: there is no scalar warp.  Every one of the 8 warps of a CTA
//   1. updates its rows (f_j += c_u K_uj + c_l K_lj) and finds its row candidates,
//   2. meets the other warps at ONE barrier (per-warp candidates -> the CTA candidate),
//   3. (warp 0 only) stores the CTA record into every CTA's mailbox of the cluster
//      (distributed shared memory; 16-byte words carrying a sequence number + checksum),
//   4. polls the G records of its own CTA's mailbox, selects (i_up, i_low) (lexicographic,
//      identical in every warp and CTA), reads the winners' alphas, labels and bit rows
//      from their records, and computes K_ul and the pair update itself (redundantly, in
//      registers),
//   5. the threads owning rows u / l of this CTA update alpha and the flags of those rows.
// So the per-iteration critical path is: row pass -> 1 CTA barrier -> one DSMEM hop ->
// a few warp reductions -> the fp64 pair update, with no warp-to-warp hand-offs.
//
// Layout (dynamic shared memory, sizes computed by bincl_smem_bytes on the host):
//   ShB header | ktab[32 W + 1] | f_s[cap] | a_s[cap] | fl_s[cap] | xb[cap][Wp] u32 |
//   cmb[2][G][RW] uint4 (the mailbox: parity, source CTA, record word)
// Row j of the CTA is handled by thread j % 256 for the whole solve (it also owns the
// row's alpha / flag updates, so they need no barrier).
#pragma once

namespace svmk {

constexpr int NTB = 256;              // threads per CTA (8 warps)
constexpr int BINCL_MAXW = 8;         // bit-row words kept in registers (d <= 256)

struct ShB {
    double exp_tab[svmexp::EXP_TABLE_DOUBLES];
    unsigned long long red_k[2][2][NTB / 32];   // [parity][up, low][warp]
    unsigned red_i[2][2][NTB / 32];
    uint4 wrec[2][NTB / 32][16];                // [parity][warp][word]: each warp's record words
};

__host__ __device__ inline size_t bincl_align(size_t x, size_t a) { return (x + a - 1) & ~(a - 1); }

// Shared-memory bytes of smo_bincl (must match the kernel's carving below).
__host__ __device__ inline size_t bincl_smem_bytes(int cap, int W, int G, int RW) {
    const int Wp = (W + 3) & ~3;
    size_t off = bincl_align(sizeof(ShB), 128);
    off += (size_t)(32 * W + 1) * 8;
    off = bincl_align(off, 16);
    off += (size_t)cap * 8 * 2 + (size_t)cap;
    off = bincl_align(off, 16);
    off += (size_t)cap * Wp * 4;
    off = bincl_align(off, 16);
    off += (size_t)2 * G * RW * 16;
    return off;
}

__device__ __forceinline__ int csa_popc4(uint32_t a, uint32_t b, uint32_t c, uint32_t e) {
    const uint32_t s1 = a ^ b ^ c;
    const uint32_t c1 = (a & b) | (c & (a ^ b));
    const uint32_t s2 = s1 ^ e, c2 = s1 & e;
    return __popc(s2) + 2 * (__popc(c1) + __popc(c2));
}

template <int KERNEL>
__global__ void __launch_bounds__(NTB, 1) smo_bincl(const Params P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    ShB& sh = *reinterpret_cast<ShB*>(smem_raw);
    const int W = P.bin_words, Wp = (W + 3) & ~3, Wq = Wp >> 2;
    const int G = P.ctas_per_rank, RW = P.crw, rw = (W + 2) / 3;
    const int cap = P.state_cap;
    size_t off = bincl_align(sizeof(ShB), 128);
    double* ktab = reinterpret_cast<double*>(smem_raw + off); off += (size_t)(32 * W + 1) * 8;
    off = bincl_align(off, 16);
    double* f_s = reinterpret_cast<double*>(smem_raw + off); off += (size_t)cap * 8;
    double* a_s = reinterpret_cast<double*>(smem_raw + off); off += (size_t)cap * 8;
    uint8_t* fl_s = smem_raw + off; off += (size_t)cap;
    off = bincl_align(off, 16);
    uint4* xb = reinterpret_cast<uint4*>(smem_raw + off); off += (size_t)cap * Wp * 4;
    off = bincl_align(off, 16);
    uint4* cmb = reinterpret_cast<uint4*>(smem_raw + off);

    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int rank = P.rank_base + blockIdx.x / G;
    const int cta = blockIdx.x % G;
    const int n_r = P.n_rows[rank];
    const int r0 = (int)(((long long)n_r * cta) / G);
    const int r1 = (int)(((long long)n_r * (cta + 1)) / G);
    const int R = r1 - r0;
    const long long gbase = P.row_off[rank] + r0;
    const double C = P.C;
    const double INF = __longlong_as_double(0x7ff0000000000000ll);

    // ---- state, resident bit rows, K table, empty mailbox
    for (int j = t; j < R; j += NTB) {
        f_s[j] = P.f[rank][r0 + j];
        a_s[j] = P.alpha[rank][r0 + j];
        fl_s[j] = P.flags[rank][r0 + j];
    }
    {
        const uint4* src = reinterpret_cast<const uint4*>(P.xblk[rank] + (long long)cta * P.cta_stride);
        for (int e = t; e < R * Wq; e += NTB) xb[e] = src[e];
    }
    for (int e = t; e < svmexp::EXP_TABLE_DOUBLES; e += NTB) sh.exp_tab[e] = svmexp::table_entry(e);
    for (int e = t; e < 2 * G * RW; e += NTB) cmb[e] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    {
        const svmexp::PtrTab tab{sh.exp_tab};
        for (int e = t; e <= 32 * W; e += NTB)
            ktab[e] = KERNEL == 1 ? svmexp::exp_cr_t(-(P.gamma * (double)e), tab) : (double)e;
    }
    __syncthreads();
    cluster_sync_all();                  // every mailbox is empty before any record lands

    Ctl* ctl = P.ctl[rank];
    long long it = ctl->it;
    long long seq = ctl->seq;
    const long long it_start = it;
    const long long max_iter = P.max_iter;
    int final_state = ST_RUNNING;
    double fu = INF, fl = -INF;
    int iu = INT_MAX, il = INT_MAX;

    bool have_update = false;            // the first pass selects from the current state
    uint32_t pu[BINCL_MAXW], pl[BINCL_MAXW];
#pragma unroll
    for (int k = 0; k < BINCL_MAXW; ++k) { pu[k] = 0u; pl[k] = 0u; }
    double cu = 0.0, cl = 0.0;
    int yu = 0, yl = 0;                  // the selected pair's labels and alphas (pending update)
    double au = 0.0, al = 0.0;
    const int nq = (R + NTB - 1) / NTB;  // rows per thread (upper bound)
    const bool trace_on = P.trace != nullptr && cta == 0 && rank == 0;
    int progress_left = 1;               // the host-visible progress word, every check_interval

    // ---- pair update (a2) of the pair selected last iteration (it - 1), in every warp: eta,
    // clipped step, snapped alphas; the owners of rows u and l update them.  Called inside
    // the row pass between the popcounts and the first use of c_u, c_l (and of the owners'
    // flags), so its serial fp64 chain overlaps the POPC-bound distance work.
    auto pair_update = [&]() {
        double Kuu, Kll, Kul;
        {
            int cuu = 0, cll = 0, cul = 0, cx = 0;
#pragma unroll
            for (int k = 0; k < BINCL_MAXW; ++k) {
                cuu += __popc(pu[k]); cll += __popc(pl[k]);
                cul += __popc(pu[k] & pl[k]); cx += __popc(pu[k] ^ pl[k]);
            }
            if (KERNEL == 1) { Kuu = 1.0; Kll = 1.0; Kul = (iu == il) ? 1.0 : ktab[cx]; }
            else { Kuu = (double)cuu; Kll = (double)cll; Kul = (double)cul; }
        }
        const double eta = Kuu + Kll - 2.0 * Kul;
        const double gap = fl - fu;
        const double yu_d = (double)yu, yl_d = (double)yl;
        const double tu = (yu == 1) ? C - au : au;
        const double tl = (yl == 1) ? al : C - al;
        double tt = gap / (eta > 1e-12 ? eta : 1e-12);
        if (tu < tt) tt = tu;
        if (tl < tt) tt = tl;
        const double au2 = (tt == tu) ? (yu == 1 ? C : 0.0) : au + yu_d * tt;
        const double al2 = (tt == tl) ? (yl == 1 ? 0.0 : C) : al - yl_d * tt;
        cu = yu_d * (au2 - au);
        cl = yl_d * (al2 - al);
        // the owners of rows u and l (thread j % NTB of the owning CTA) update them before
        // their next row pass
        {
            const int lu = (int)((long long)iu - gbase), ll = (int)((long long)il - gbase);   // |.| < 2^31
            const bool own_u = (unsigned)lu < (unsigned)R && (lu & (NTB - 1)) == t;
            const bool own_l = (unsigned)ll < (unsigned)R && (ll & (NTB - 1)) == t;
            if (own_u) { a_s[lu] = au2; fl_s[lu] = flags_of(yu, au2, C); }
            if (own_l) { a_s[ll] = al2; fl_s[ll] = flags_of(yl, al2, C); }
        }
        if (--progress_left == 0) {
            progress_left = P.check_interval;
            if (t == 0 && cta == 0 && rank == 0 && P.progress)
                *(volatile unsigned long long*)P.progress = (unsigned long long)(it - 1);
        }
        if (trace_on && t == 0 && it - 1 < P.trace_cap) { P.trace[2 * (it - 1)] = iu; P.trace[2 * (it - 1) + 1] = il; }
    };
    const bool timing = P.timers != nullptr && blockIdx.x == 0 && t == 0;
    unsigned long long ph_acc[PH_N] = {};
    long long ph_t = clock64();
#define BPHASE(ph) do { if (timing) { const long long c_ = clock64(); ph_acc[ph] += (unsigned long long)(c_ - ph_t); ph_t = c_; } } while (0)
    for (;;) {
        // ================= row pass: f update (a3-a5) and this thread's candidates
        double bfu = INF, bfl = -INF;
        int bju = INT_MAX, bjl = INT_MAX;
        constexpr int BT = 8;
        for (int q0 = 0; q0 < nq; q0 += BT) {
            double fj[BT];
            uint8_t gq[BT];
            int jq[BT];
#pragma unroll
            for (int q = 0; q < BT; ++q) jq[q] = min((q0 + q) * NTB + t, R - 1);
            if (have_update) {
                int du[BT], dl[BT];
#pragma unroll
                for (int q = 0; q < BT; ++q) { du[q] = 0; dl[q] = 0; }
#pragma unroll
                for (int w4 = 0; w4 < BINCL_MAXW / 4; ++w4) {
                    if (w4 < Wq) {
                        uint4 xv[BT];
#pragma unroll
                        for (int q = 0; q < BT; ++q) xv[q] = xb[jq[q] * Wq + w4];
                        const uint32_t u0 = pu[4 * w4], u1 = pu[4 * w4 + 1], u2 = pu[4 * w4 + 2], u3 = pu[4 * w4 + 3];
                        const uint32_t l0 = pl[4 * w4], l1 = pl[4 * w4 + 1], l2 = pl[4 * w4 + 2], l3 = pl[4 * w4 + 3];
#pragma unroll
                        for (int q = 0; q < BT; ++q) {
                            if (KERNEL == 1) {
                                // popcount of 4 words with a carry-save step (3 POPC instead of
                                // 4; POPC is the row pass's busiest pipe): a + b + c = s1 + 2 c1,
                                // s1 + e = s2 + 2 c2  =>  sum = popc(s2) + 2 (popc(c1) + popc(c2))
                                du[q] += csa_popc4(xv[q].x ^ u0, xv[q].y ^ u1, xv[q].z ^ u2, xv[q].w ^ u3);
                                dl[q] += csa_popc4(xv[q].x ^ l0, xv[q].y ^ l1, xv[q].z ^ l2, xv[q].w ^ l3);
                            } else {
                                du[q] += csa_popc4(xv[q].x & u0, xv[q].y & u1, xv[q].z & u2, xv[q].w & u3);
                                dl[q] += csa_popc4(xv[q].x & l0, xv[q].y & l1, xv[q].z & l2, xv[q].w & l3);
                            }
                        }
                    }
                }
                if (q0 == 0) pair_update();      // c_u, c_l; owners' alpha / flags
                double ku[BT], kl[BT];
#pragma unroll
                for (int q = 0; q < BT; ++q) {
                    ku[q] = ktab[du[q]];      // RBF: K(x_j, x_j) = ktab[0] = 1 (R16)
                    kl[q] = ktab[dl[q]];
                    // rows past the end (clamped to R - 1, whose owner may be updating it)
                    // are not read: their results are discarded anyway
                    const bool in = (q0 + q) * NTB + t < R;
                    fj[q] = in ? f_s[jq[q]] : 0.0;
                    gq[q] = in ? fl_s[jq[q]] : (uint8_t)0;
                }
#pragma unroll
                for (int q = 0; q < BT; ++q) {
                    fj[q] = fma(cl, kl[q], fma(cu, ku[q], fj[q]));
                    if ((q0 + q) * NTB + t < R) f_s[jq[q]] = fj[q];
                }
            } else {
#pragma unroll
                for (int q = 0; q < BT; ++q) {
                    const bool in = (q0 + q) * NTB + t < R;
                    fj[q] = in ? f_s[jq[q]] : 0.0;
                    gq[q] = in ? fl_s[jq[q]] : (uint8_t)0;
                }
            }
            double cfu[BT], cfl[BT];
            int cju[BT], cjl[BT];
#pragma unroll
            for (int q = 0; q < BT; ++q) {
                const bool ok = (q0 + q) * NTB + t < R;
                cfu[q] = (ok && (gq[q] & FL_UP)) ? fj[q] : INF;
                cfl[q] = (ok && (gq[q] & FL_LOW)) ? fj[q] : -INF;
                cju[q] = (q0 + q) * NTB + t; cjl[q] = cju[q];
            }
            // rows increase with q: on equal f the lower q wins; a tie with the running best
            // (earlier rows) keeps the running best
#pragma unroll
            for (int s2 = 1; s2 < BT; s2 <<= 1)
#pragma unroll
                for (int q = 0; q + s2 < BT; q += 2 * s2) {
                    if (cfu[q + s2] < cfu[q]) { cfu[q] = cfu[q + s2]; cju[q] = cju[q + s2]; }
                    if (cfl[q + s2] > cfl[q]) { cfl[q] = cfl[q + s2]; cjl[q] = cjl[q + s2]; }
                }
            if (cfu[0] < bfu) { bfu = cfu[0]; bju = cju[0]; }
            if (cfl[0] > bfl) { bfl = cfl[0]; bjl = cjl[0]; }
        }
        BPHASE(PH_C_DIST);
        ++seq;
        const int par = (int)(seq & 1);
        const uint32_t sq = (uint32_t)seq & 0xffffu;
        {
            unsigned long long kwu, kwl;
            unsigned iwu, iwl;
            argmin_redux(0xffffffffu, bju == INT_MAX ? ~0ull : fkey(bfu), (unsigned)bju, kwu, iwu);
            argmin_redux(0xffffffffu, bjl == INT_MAX ? ~0ull : ~fkey(bfl), (unsigned)bjl, kwl, iwl);
            if (lane == 0) {
                sh.red_k[par][0][warp] = kwu; sh.red_i[par][0][warp] = iwu;
                sh.red_k[par][1][warp] = kwl; sh.red_i[par][1][warp] = iwl;
            }
            // this warp's record words (word h = lane): 0 (i_up, f_up), 1 (i_low, f_low),
            // 2 (y_up | y_low << 16, a_up), 3 (0, a_low), 4.. the candidates' bit rows.
            // Built before the barrier, so after it the CTA record is a copy.
            const int ju = (int)iwu, jl = (int)iwl;
            const bool eu = ju == INT_MAX, el = jl == INT_MAX;
            const int juc = eu ? 0 : ju, jlc = el ? 0 : jl;
            const double au_c = a_s[juc], al_c = a_s[jlc];
            const uint8_t gu_c = fl_s[juc], gl_c = fl_s[jlc];
            const int yu_ = eu ? 0 : ((gu_c & FL_POS) ? 1 : -1);
            const int yl_ = el ? 0 : ((gl_c & FL_POS) ? 1 : -1);
            const int hr = lane - 4;                          // row word index (lanes >= 4)
            const bool is_u = hr < rw;
            const int k0 = max(3 * (hr - (is_u ? 0 : rw)), 0);
            const bool er = is_u ? eu : el;
            const uint32_t* row = reinterpret_cast<const uint32_t*>(xb) + (size_t)(is_u ? juc : jlc) * Wp;
            const uint32_t e0 = row[min(k0, Wp - 1)], e1 = row[min(k0 + 1, Wp - 1)], e2 = row[min(k0 + 2, Wp - 1)];
            const uint32_t r0w = (!er && k0 < W) ? e0 : 0u;
            const uint32_t r1w = (!er && k0 + 1 < W) ? e1 : 0u;
            const uint32_t r2w = (!er && k0 + 2 < W) ? e2 : 0u;
            const uint32_t a = lane == 0 ? (eu ? 0xffffffffu : (uint32_t)(gbase + ju))
                             : lane == 1 ? (el ? 0xffffffffu : (uint32_t)(gbase + jl))
                             : lane == 2 ? (uint32_t)((yu_ & 0xffff) | (yl_ << 16))
                             : lane == 3 ? 0u : r0w;
            const double vd = lane == 0 ? (eu ? INF : fkey_inv(kwu))
                            : lane == 1 ? (el ? -INF : fkey_inv(~kwl))
                            : lane == 2 ? (eu ? 0.0 : au_c) : (el ? 0.0 : al_c);
            const unsigned long long v = lane < 4 ? (unsigned long long)__double_as_longlong(vd)
                                                  : ((unsigned long long)r1w | ((unsigned long long)r2w << 32));
            if (lane < RW) sh.wrec[par][warp][lane] = rec_pack(sq, a, v);
        }
        BPHASE(PH_C_REDUCE);
        __syncthreads();                 // the one CTA barrier of the iteration
        (void)*(volatile unsigned*)&sh.red_i[par][0][0];
        BPHASE(PH_C_WAITB);

        // ================= exchange seq (a6).  Control flow is warp-uniform throughout
        // (divergent branches cost more than the arithmetic here): lanes compute with
        // clamped indices and select.
        {
            // every warp forms the CTA candidate and copies its record from the winning
            // warps' words; warp w stores it into the CTAs j = w, w + 8, ... (one store
            // instruction per target: a DSMEM store instruction costs ~27 cycles per
            // destination CTA)
            const bool in8 = lane < NTB / 32;
            const int l8 = lane & (NTB / 32 - 1);
            unsigned long long kmu, kml;
            unsigned jmu, jml;
            argmin_redux(0xffffffffu, in8 ? sh.red_k[par][0][l8] : ~0ull, in8 ? sh.red_i[par][0][l8] : 0xffffffffu, kmu, jmu);
            argmin_redux(0xffffffffu, in8 ? sh.red_k[par][1][l8] : ~0ull, in8 ? sh.red_i[par][1][l8] : 0xffffffffu, kml, jml);
            // row j belongs to warp (j mod 256) / 32
            const int wu = (int)jmu == INT_MAX ? 0 : (int)((jmu & (NTB - 1)) >> 5);
            const int wl = (int)jml == INT_MAX ? 0 : (int)((jml & (NTB - 1)) >> 5);
            const int h = min(lane, RW - 1);
            const bool from_u = h == 0 || h == 2 || (h >= 4 && h - 4 < rw);
            uint4 wv = sh.wrec[par][from_u ? wu : wl][h];
            if (h == 2) {                                 // y_up from u's warp, y_low from l's
                const uint4 w2l = sh.wrec[par][wl][2];
                wv = rec_pack(sq, (rec_aux(wv) & 0xffffu) | (rec_aux(w2l) & 0xffff0000u), rec_payload(wv));
            }
            const uint32_t src = smem_u32(cmb + ((size_t)par * G + cta) * RW + h);
            for (int j = warp; j < G; j += NTB / 32) {
                uint32_t ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(src), "r"(j));
                if (lane < RW) st_cluster_v4(ra, wv);
            }
        }
        BPHASE(PH_S_PUBLISH);
        // every warp: lanes 0-15 poll word 0 (up candidate), lanes 16-31 word 1 (low) of the
        // records of CTAs 0..G-1 (lanes past G re-read the last record)
        const bool lowh = lane >= 16;
        const int hl = lane & 15;
        const uint4* rp = cmb + ((size_t)par * G + min(hl, G - 1)) * RW + (lowh ? 1 : 0);
        uint4 w;
        bool to = false;
        {
            long long t0 = 0;
            unsigned int spins = 0;
            for (;;) {
                w = ld_volatile_shared_v4(rp);
                if (__all_sync(0xffffffffu, rec_ok(w, sq))) break;
                if (P.poll_ns > 0) __nanosleep(P.poll_ns);   // (tuning: poll backoff)
                if ((++spins & 255u) == 0) {
                    const long long now = globaltimer();
                    if (t0 == 0) t0 = now;
                    else if (now - t0 > P.timeout_ns) { to = true; break; }
                }
            }
        }
        const bool tmo = __any_sync(0xffffffffu, to);
        BPHASE(PH_S_POLL);
        const unsigned pi = (hl < G) ? rec_aux(w) : 0xffffffffu;
        const unsigned long long k0w = pi == 0xffffffffu ? ~0ull : fkey(rec_f64(w));
        const unsigned long long kup = lowh ? ~0ull : k0w;
        const unsigned long long klo = lowh ? (pi == 0xffffffffu ? ~0ull : ~k0w) : ~0ull;
        unsigned long long kwu, kwl;
        unsigned iwu, iwl;
        argmin_redux(0xffffffffu, kup, lowh ? 0xffffffffu : pi, kwu, iwu);
        argmin_redux(0xffffffffu, klo, lowh ? pi : 0xffffffffu, kwl, iwl);
        const unsigned hu = __ballot_sync(0xffffffffu, !lowh && pi == iwu && kup == kwu) & 0xffffu;
        const unsigned hlw = __ballot_sync(0xffffffffu, lowh && pi == iwl && klo == kwl) >> 16;
        iu = iwu == 0xffffffffu ? INT_MAX : (int)iwu;
        il = iwl == 0xffffffffu ? INT_MAX : (int)iwl;
        fu = iu == INT_MAX ? INF : fkey_inv(kwu);
        fl = il == INT_MAX ? -INF : fkey_inv(~kwl);
        const int rec_u = hu ? __ffs(hu) - 1 : 0, rec_l = hlw ? __ffs(hlw) - 1 : 0;
        int dec = ST_RUNNING;
        if (tmo) dec = ST_TIMEOUT;
        else if (iu == INT_MAX || il == INT_MAX) dec = ST_CONVERGED;
        else if (fl - fu <= 2.0 * P.tol) dec = ST_CONVERGED;
        else if (it == max_iter) dec = ST_MAXITER;
        else if (P.iter_limit > 0 && it - it_start == P.iter_limit) dec = ST_LIMIT;
        if (dec != ST_RUNNING) { final_state = dec; break; }
        BPHASE(PH_S_READ);

        // ---- the winners' alpha / label (words 2, 3) and bit rows (words 4..) -- lane 0:
        // w2 of u's record, 1: w2 of l's, 2: w3 of l's, 3..3+rw-1: u's row, then l's row
        // (other lanes re-read lane 0's word)
        const int nwl = 3 + 2 * rw;
        const int ln = lane < nwl ? lane : 0;
        const int rr = (ln == 0 || (ln >= 3 && ln < 3 + rw)) ? rec_u : rec_l;
        const int hh = ln < 3 ? (ln == 2 ? 3 : 2) : (ln < 3 + rw ? 4 + (ln - 3) : 4 + rw + (ln - 3 - rw));
        const uint4* wp = cmb + ((size_t)par * G + rr) * RW + hh;
        uint4 wa = ld_volatile_shared_v4(wp);
        {
            unsigned int spins = 0;
            while (!__all_sync(0xffffffffu, rec_ok(wa, sq))) {   // (almost) never taken
                wa = ld_volatile_shared_v4(wp);
                if (++spins > (1u << 24)) break;
            }
        }
        const uint32_t wa_aux = rec_aux(wa), wa_lo = rec_lo(wa), wa_hi = rec_hi(wa);
        yu = (int)(int16_t)(__shfl_sync(0xffffffffu, wa_aux, 0) & 0xffffu);
        au = __hiloint2double((int)__shfl_sync(0xffffffffu, wa_hi, 0), (int)__shfl_sync(0xffffffffu, wa_lo, 0));
        yl = (int)(int16_t)(__shfl_sync(0xffffffffu, wa_aux, 1) >> 16);
        al = __hiloint2double((int)__shfl_sync(0xffffffffu, wa_hi, 2), (int)__shfl_sync(0xffffffffu, wa_lo, 2));
#pragma unroll
        for (int k = 0; k < BINCL_MAXW; ++k) {
            const int su = 3 + k / 3, sl = 3 + rw + k / 3;
            // a row word triple travels as (aux, payload lo, payload hi)
            const uint32_t cu_ = (k % 3 == 0) ? wa_aux : ((k % 3 == 1) ? wa_lo : wa_hi);
            const uint32_t vu = __shfl_sync(0xffffffffu, cu_, su & 31);
            const uint32_t vl = __shfl_sync(0xffffffffu, cu_, sl & 31);
            pu[k] = k < W ? vu : 0u;
            pl[k] = k < W ? vl : 0u;
        }
        BPHASE(PH_S_PIVOT);
        BPHASE(PH_S_KUL);
        have_update = true;
        ++it;
    }
#undef BPHASE
    if (timing)
        for (int k = 0; k < PH_N; ++k) atomicAdd(&P.timers[k], ph_acc[k]);

    // ---- write back (the pending update of the last selection is not applied: the loop
    // ends at a selection, exactly as the smo_persistent kernel does)
    __syncthreads();
    for (int j = t; j < R; j += NTB) {
        P.f[rank][r0 + j] = f_s[j];
        P.alpha[rank][r0 + j] = a_s[j];
        P.flags[rank][r0 + j] = fl_s[j];
    }
    if (t == 0 && cta == 0) {
        ctl->it = it;
        ctl->seq = seq;
        ctl->state = final_state;
        ctl->b_up = fu;
        ctl->b_low = fl;
        ctl->i_up = iu == INT_MAX ? -1 : iu;
        ctl->i_low = il == INT_MAX ? -1 : il;
    }
    __syncwarp();
    cluster_sync_all();                  // no CTA leaves while a peer may address its mailbox
}

}  // namespace svmk
