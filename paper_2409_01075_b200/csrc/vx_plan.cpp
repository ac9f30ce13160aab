// vx_plan.cpp -- the offline strategy table and the runtime analytical selector of Vortex
// (arXiv 2409.01075) for sm_100a.  Host-only C++, no CUDA calls: a plan built with
// vx_plan_ex and a captured descriptor can be planned and selected on a CPU-only host.
//
//   vx_plan         Alg. 2 "Candidates Generation Algorithm":
//                   L0 InitCands -> FilterByISA; L>=1 InitCands -> FilterByMultiples + map,
//                   over the sm_100a hierarchy of DESIGN.md 3.1:
//                     L0 tcgen05.mma.kind::f16 instruction tile (UM x UN x 16)
//                     L1 TMEM accumulator (UM lanes x AN fp32 columns x acc_stages)
//                     L2 CTA tile in SMEM (BM x BN x 64, S-stage TMA ring)
//                     L3 grid schedule (operand swap, K-split s over a CTA cluster)
//   vx_plan_select  Eqs. 2-4 evaluated per (rung, split) for the
//                   runtime shape in integer cycles, argmin Eq. 1,
//                   grid configuration.  DESIGN.md 3.3 is the spec; the
//                   readings R1-R14 it lists are cited inline.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <set>
#include <string>
#include <tuple>

#include "vx_internal.h"

namespace vx {

bool kernel_available(int family, int bm, int bn, int mc = 1, int occ = 1);  // vx_dispatch.cu

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int in_bytes(vx_dtype d) { return d == VX_FP32 ? 4 : 2; }
int out_bytes(vx_dtype d) { return d == VX_FP32 ? 4 : 2; }

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- Eqs. 2-4 --------------------------------------------------------------------------
// T_Load / T_Store = bytes moved / bandwidth of that layer, ceiling (R14)
static inline int64_t t_move(int64_t bytes, int64_t bw_milli) { return cdiv(bytes * 1000, bw_milli); }
// Eq. 2: T_Load + (trips-1) max(T_Load, Cost_{L-1}) + Cost_{L-1} + T_Store
static inline int64_t eq2(int64_t tl, int64_t trips, int64_t inner, int64_t ts) {
    return tl + (trips - 1) * std::max(tl, inner) + inner + ts;
}
// Eq. 3: ceil(sizeof(ParallelLoop) / |HardwareUnit|)
static inline int64_t eq3(int64_t extent, int64_t units) { return cdiv(extent, units); }

// ---- Alg. 2 over the sm_100a levels -----------------------------------------------------
namespace {

struct L0 { int um, un, uk; };
struct L1 { int am, an, st; };
struct L2 { int bm, bn, bk, S, st, occ; };

const int kUmLattice[] = {64, 128, 256};                  // R1
const int kNLattice[] = {8, 16, 32, 64, 128, 192, 256};   // R1

// tcgen05.mma.kind::f16 legality (PTX ISA shape table)
bool isa_ok(const L0& c) {
    if (c.uk != kUmmaK) return false;
    if (c.um == 64) return c.un % 8 == 0 && c.un >= 8 && c.un <= 256;
    if (c.um == 128 || c.um == 256) return c.un % 16 == 0 && c.un >= 16 && c.un <= 256;
    return false;
}

// FilterByMultiples: for prev in prevCands, for each candidate that is an integer multiple
// of prev: keep it (first-insertion order) and record the link.
template <class C, class P, class Div>
std::vector<C> sieve(const std::vector<C>& cands, const std::vector<P>& prev, Div divides,
                     int64_t* links) {
    std::vector<C> out;
    std::vector<char> taken(cands.size(), 0);
    int64_t nl = 0;
    for (const P& p : prev)
        for (size_t i = 0; i < cands.size(); ++i)
            if (divides(p, cands[i])) {
                ++nl;
                if (!taken[i]) { taken[i] = 1; out.push_back(cands[i]); }
            }
    if (links) *links = nl;
    return out;
}

const char* family_name(int f) {
    return f == kUmma ? "umma" : f == kUmmaSwap ? "umma_swap" : f == kSimt ? "simt" : "gemv";
}

}  // namespace

static vx_status build_rungs(vx_plan_s* p) {
    const vx_device_desc& d = p->desc;
    std::vector<Rung> rungs;
    if (p->in == VX_BF16 || p->in == VX_FP16) {
        const int in_b = 2;
        // L0: InitCands = lattice; FilterByISA
        std::vector<L0> l0;
        for (int um : kUmLattice)
            for (int un : kNLattice) {
                L0 c{um, un, kUmmaK};
                if (isa_ok(c)) l0.push_back(c);
            }
        // L1: TMEM accumulators within the column capacity (R2: no window on TMEM)
        std::vector<L1> l1i;
        for (int am : kUmLattice)
            for (int an : kNLattice)
                for (int st = 1; st <= 2; ++st)
                    if (st * an <= d.tmem_cols) l1i.push_back({am, an, st});
        std::vector<L1> l1 = sieve(l1i, l0, [](const L0& a, const L1& c) {
            return c.am == a.um && c.an % a.un == 0; }, nullptr);
        // L2: CTA tiles; stage count = deepest ring that fits SMEM; window [1/8, 1] (R3, R5)
        std::vector<L2> l2i;
        for (const L1& a : l1) {
            int cg = a.am == 256 ? 2 : 1;
            int64_t stage = (int64_t)(a.am / cg + a.an / cg) * kBkTc * in_b;
            int64_t fit = (d.smem_optin - kSmemReserve - kEpiStaging) / stage;
            int S = (int)std::min<int64_t>(kMaxStages, fit);
            if (S < 2) continue;
            int64_t foot = S * stage + kSmemReserve + kEpiStaging;
            if (foot * 8 < d.smem_optin) continue;
            l2i.push_back({a.am, a.an, kBkTc, S, a.st, 1});
            // occupancy-2 ring (R5b): sized so two CTAs share an SM -- half the SM's shared
            // memory each (less the per-CTA system reserve) and half its TMEM columns -- so a
            // launch's CTAs become resident while the previous grid still runs
            if (cg == 1 && 2 * a.st * a.an <= d.tmem_cols) {
                int64_t fit2 = (d.smem_per_sm / 2 - kCtaSysSmem - kSmemReserve - kEpiStagingLean) / stage;
                int S2 = (int)std::min<int64_t>(kMaxStages, fit2);
                int64_t foot2 = S2 * stage + kSmemReserve + kEpiStagingLean;
                if (S2 >= 2 && S2 < S && foot2 * 8 >= d.smem_optin)
                    l2i.push_back({a.am, a.an, kBkTc, S2, a.st, 2});
            }
        }
        std::vector<L2> l2 = sieve(l2i, l1, [](const L1& a, const L2& c) {
            return c.bm % a.am == 0 && c.bn % a.an == 0 && c.st == a.st && c.bk % kUmmaK == 0; },
            nullptr);
        // L3: grid schedules over implemented kernels (R6), splits dividing the k-blocks (R7)
        const int64_t kb = cdiv(p->K, kBkTc);
        for (const L2& c : l2) {
            int cg = c.bm == 256 ? 2 : 1;
            for (int swap = 0; swap <= 1; ++swap) {
                int fam = swap ? kUmmaSwap : kUmma;
                if (cg == 2 && swap) continue;      // pair rungs are non-swapped
                // a pair CTA holding fewer than 64 B rows needs B K-major (VX_B_NK): the
                // MN-major 128-B swizzle atom (B stored K x N) is 64 elements wide
                if (cg == 2 && c.bn / 2 < 64 && p->bl != VX_B_NK) continue;
                int64_t stage = (int64_t)(c.bm / cg + c.bn / cg) * c.bk * in_b;
                // TMA-multicast clusters of mc CTAs sharing the A tile: the
                // multicast sub-box (A rows / mc) must be whole 8-row swizzle atoms and a
                // packed B keeps its own 5-D load path, so multicast needs B unpacked
                for (int mc : {1, 2, 4}) {
                    if (c.st != 2 || !kernel_available(fam, c.bm, c.bn, mc, c.occ)) continue;
                    if (c.occ == 2 && mc > 1) continue;   // lean CTAs are not clustered
                    if (mc > 1 && (cg > 1 || (swap ? c.bn : c.bm) / mc % 8 != 0 ||
                                   p->bl == VX_B_PACKED))
                        continue;
                    Rung r{};
                    r.family = fam; r.cg = cg; r.um = c.bm; r.un = c.bn; r.acc_stages = c.st;
                    r.bm = c.bm; r.bn = c.bn; r.bk = c.bk; r.stages = c.S; r.swap = swap;
                    r.mc = mc;
                    r.occ = c.occ;
                    if (mc > 1 || c.occ == 2) {   // multicast clusters and lean CTAs run
                        r.splits = {1};           // the persistent schedule
                        rungs.push_back(r);
                        continue;
                    }
                    if (mc > 1) {
                        r.splits = {1};     // multicast clusters run the persistent schedule
                        rungs.push_back(r);
                        continue;
                    }
                    for (int s : {1, 2, 4, 8}) {
                        if (kb % s != 0 || s * cg > kClusterMax) continue;
                        if (s > 1 && (cg > 1 || (int64_t)c.bm * (c.bn + 4) * 4 > c.S * stage)) continue;
                        r.splits.push_back(s);
                    }
                    r.splits.push_back(0);  // stream-K over (tile, k-block) units (R19)
                    rungs.push_back(r);
                }
            }
        }
        // adaptive backend (R20): CUDA-core GEMV-style rungs for tiny M (M <= MT), competing
        // in the same argmin; not for pre-packed weights
        if (p->bl != VX_B_PACKED)
            for (int mt : {1, 2, 4, 8}) {
                if (!kernel_available(kGemv, mt, kGemvColsPerCta)) continue;
                Rung r{};
                r.family = kGemv; r.cg = 1; r.um = 1; r.un = 1; r.acc_stages = 1;
                r.bm = mt; r.bn = kGemvColsPerCta; r.bk = kGemvBk; r.stages = 1; r.swap = 0;
                r.mc = 1; r.occ = 1;
                r.splits = {1};
                rungs.push_back(r);
            }
        p->counts = {(int64_t)l0.size(), (int64_t)l1.size(), (int64_t)l2.size(), (int64_t)rungs.size()};
    } else {
        // CUDA-core mode: L0 FFMA thread tiles, L2 CTA tiles (BK = 16)
        struct T { int bm, bn, tm, tn; };
        const T tiles[] = {{32, 32, 2, 4}, {64, 64, 4, 4}, {128, 64, 8, 4}};
        std::set<std::pair<int, int>> l0;
        for (const T& t : tiles) l0.insert({t.tm, t.tn});
        int64_t n2 = 0;
        for (const T& t : tiles) {
            int threads = (t.bm / t.tm) * (t.bn / t.tn);
            if (threads > d.max_threads_per_block) continue;
            if (t.bm % t.tm || t.bn % t.tn) continue;
            ++n2;
            if (!kernel_available(kSimt, t.bm, t.bn)) continue;
            Rung r{};
            r.family = kSimt; r.cg = 1; r.um = t.tm; r.un = t.tn; r.acc_stages = 1;
            r.bm = t.bm; r.bn = t.bn; r.bk = kSimtBk; r.stages = 2; r.swap = 0;
            r.mc = 1; r.occ = 1;
            r.splits = {1};
            rungs.push_back(r);
        }
        p->counts = {(int64_t)l0.size(), (int64_t)l0.size(), n2, (int64_t)rungs.size()};
    }
    // deterministic ids (R13)
    std::sort(rungs.begin(), rungs.end(), [](const Rung& a, const Rung& b) {
        return std::tie(a.family, a.bm, a.bn, a.stages, a.swap, a.mc, a.occ) <
               std::tie(b.family, b.bm, b.bn, b.stages, b.swap, b.mc, b.occ); });
    for (size_t i = 0; i < rungs.size(); ++i) {
        Rung& r = rungs[i];
        r.rung_id = (int32_t)i;
        char key[64];
        if (r.occ == 2) snprintf(key, sizeof key, "%s_o2_%dx%d", family_name(r.family), r.bm, r.bn);
        else if (r.mc > 1) snprintf(key, sizeof key, "%s_mc%d_%dx%d", family_name(r.family), r.mc, r.bm, r.bn);
        else snprintf(key, sizeof key, "%s_%dx%d", family_name(r.family), r.bm, r.bn);
        const RungConst* c = p->cal.find(key);
        if (!c) { set_error("no calibration for rung %s", key); return VX_ERR_UNSUPPORTED; }
        r.mac_milli = c->mac_milli; r.l2s_milli = c->l2s_milli;
        r.epi_milli = c->epi_milli; r.fixed = c->fixed;
    }
    if (rungs.empty()) { set_error("strategy table is empty"); return VX_ERR_UNSUPPORTED; }
    p->rungs = std::move(rungs);
    return VX_OK;
}

// stream-K is admitted only where wave quantization is what it fixes: the data-parallel
// schedule of the rung needs at most kSkMaxWaves waves; and only where every CTA's share of
// the units is at least half a tile's K loop, so a cut tile gathers few partials (R19)
constexpr int64_t kSkMaxWaves = 3;
static bool sk_admissible(const vx_plan_s* p, const Rung& r, int64_t batch, int64_t M, int64_t N) {
    const int64_t mt = r.swap ? N : M, nt = r.swap ? M : N;
    const int64_t tiles = batch * cdiv(mt, r.bm) * cdiv(nt, r.bn);
    const int64_t act = (int64_t)p->desc.max_active_clusters[r.cg == 2 ? 1 : 0];
    const int64_t slots = act * r.cg;
    const int64_t kb = cdiv(p->K, r.bk);
    const int64_t U = tiles * kb;
    const int64_t G = act < U ? act : U;
    return tiles * r.cg <= kSkMaxWaves * slots && 2 * cdiv(U, G) >= kb;
}

// ---- runtime cost ----------------------------------------------------------
static void rung_cost(const vx_plan_s* p, const Rung& r, int s, int64_t batch, int64_t M,
                      int64_t N, vx_choice* o) {
    const vx_device_desc& d = p->desc;
    const Calib& cal = p->cal.glob;
    const int64_t K = p->K;
    const int in_b = in_bytes(p->in), out_b = out_bytes(p->out);
    const int64_t bm = r.bm, bn = r.bn, bk = r.bk;
    // padding only at the outermost level (fig:padding)
    const int64_t mt = r.swap ? N : M, nt = r.swap ? M : N;
    const int64_t tm = cdiv(mt, bm), tn = cdiv(nt, bn);
    const int64_t tiles = batch * tm * tn;
    const int64_t kb = cdiv(K, bk);
    if (r.family == kGemv) {
        // CUDA-core GEMV rung (R20): a CTA = MT rows x 8 columns; k-steps of 1024
        const int64_t tiles_g = batch * cdiv(N, bn);
        const int64_t slots_g = (int64_t)d.sm_count * kGemvOcc;
        const int64_t Fg = eq3(tiles_g, slots_g);
        const int64_t trips_g = cdiv(K, bk);
        const int64_t inner_g = t_move(bm * bn * bk, r.mac_milli);
        const int64_t ls_g = t_move(bn * bk * in_b + bm * bk * in_b, r.l2s_milli);
        const int64_t lh_g = t_move((int64_t)in_b * batch * K * (N + M), Fg * trips_g * cal.hbm_milli);
        const int64_t tl_g = std::max(ls_g, lh_g);
        const int64_t ts_g = std::max(t_move(bm * bn * out_b, r.epi_milli),
                                      t_move((int64_t)out_b * batch * M * N, Fg * cal.hbm_milli));
        o->rung_id = r.rung_id; o->split = 1; o->family = r.family; o->swap = 0;
        o->bm = r.bm; o->bn = r.bn; o->stages = r.stages;
        o->tiles_m = 1; o->tiles_n = (int32_t)cdiv(N, bn); o->grid = (int32_t)tiles_g;
        o->cluster = 1; o->mc = 1;
        o->cost = Fg * eq2(tl_g, trips_g, inner_g, ts_g) + r.fixed;
        return;
    }
    if (s == 0) {
        // stream-K (R19): G resident CTAs share U = tiles x k-blocks units evenly; one wave
        const int64_t U = tiles * kb;
        // work is split over resident CTAs, or CTA pairs for cta_group::2 rungs
        const int64_t G = std::min<int64_t>(d.max_active_clusters[r.cg == 2 ? 1 : 0], U);
        const int64_t units = cdiv(U, G);                       // temporal loop per CTA
        const int64_t segs = cdiv(units, kb) + 1;               // tile segments per CTA (bound)
        const int64_t inner = t_move(bm * bn * bk, r.mac_milli);
        const int64_t l_smem = t_move((std::min(bm, mt) + std::min(bn, nt)) * bk * in_b, r.l2s_milli);
        const int64_t l_hbm = t_move((int64_t)in_b * batch * K * (mt + nt), units * cal.hbm_milli);
        const int64_t tl = std::max(l_smem, l_hbm);
        const int64_t tm_ = eq2(tl, units, inner, 0);
        const int64_t st = std::max(t_move(bm * bn * out_b, r.epi_milli),
                                    t_move((int64_t)out_b * batch * M * N, segs * cal.hbm_milli));
        // a cut tile is finished by adding ceil(kb/units) partials (one write + read each);
        // every CTA handles its own rows (a pair's two CTAs their bm/2-row halves, in parallel)
        const int64_t fix = cdiv(kb, units) * t_move(2 * (bm / r.cg) * bn * 4, cal.skfix_milli);
        o->rung_id = r.rung_id; o->split = 0; o->family = r.family; o->swap = r.swap;
        o->bm = r.bm; o->bn = r.bn; o->stages = r.stages;
        o->tiles_m = (int32_t)tm; o->tiles_n = (int32_t)tn; o->grid = (int32_t)(G * r.cg);
        o->cluster = r.cg; o->mc = 1;
        o->cost = std::max(tm_, segs * st) + st + fix + r.fixed;
        if (G * r.cg > d.sm_count / 2) o->cost += cal.stagger;   // R21
        return;
    }
    const int64_t trips = kb / s;            // sizeof(TemporalLoop) at the CTA level (R8)
    // multicast clusters work on cluster tiles: mc consecutive tiles along the
    // axis that does NOT share the A tile (Q for non-swapped, P for swapped rungs)
    const int64_t mc = r.mc;
    const int64_t tm_c = (mc > 1 && r.swap) ? cdiv(tm, mc) * mc : tm;
    const int64_t tn_c = (mc > 1 && !r.swap) ? cdiv(tn, mc) * mc : tn;
    const int64_t W = batch * tm_c * tn_c * s * r.cg;   // sizeof(ParallelLoop) in CTAs
    int64_t slots;
    if (r.family == kSimt) {
        int64_t threads = (bm / r.um) * (bn / r.un);
        int64_t foot = 2 * (bm + bn) * bk * 4 + kSmemReserve;
        int64_t occ = std::min<int64_t>(std::min<int64_t>(d.smem_per_sm / foot,
                                        d.max_threads_per_sm / threads), 32);
        slots = (int64_t)d.sm_count * std::max<int64_t>(occ, 1);
    } else {
        const int64_t csz = s * r.cg * mc;   // CTAs per cluster
        int ci = csz == 1 ? 0 : csz == 2 ? 1 : csz == 4 ? 2 : 3;
        slots = (int64_t)d.max_active_clusters[ci] * csz;
    }
    const int64_t F = eq3(W, slots);         // Eq. 3, |HardwareUnit| = resident CTAs (R9)
    const int64_t active = std::min(W, slots);
    int64_t inner, l_smem;
    if (r.family == kSimt) {
        int64_t occ = cdiv(active, d.sm_count);
        inner = t_move(bm * bn * bk * occ, r.mac_milli);
        l_smem = t_move((bm + bn) * bk * in_b * occ, r.l2s_milli);
    } else {
        inner = t_move(bm * bn * bk, r.mac_milli);           // Cost_{L-1}
        // rows past M / N are zero-filled by TMA without memory traffic (R10); a multicast
        // cluster's CTA loads only its 1/mc share of the shared A tile (SURVEY C2 mc_A)
        const int64_t p_rows = (mc > 1 && !r.swap) ? bm / mc : std::min(bm, mt);
        const int64_t q_rows = (mc > 1 && r.swap) ? bn / mc : std::min(bn, nt);
        l_smem = t_move((p_rows + q_rows) * bk * in_b, r.l2s_milli);
    }
    const int64_t uniq = (int64_t)in_b * batch * K * (mt + nt);
    const int64_t l_hbm = t_move(uniq, F * trips * cal.hbm_milli);   // R10
    const int64_t tl = std::max(l_smem, l_hbm);                       // T_Load
    const int64_t cbytes = (int64_t)out_b * batch * M * N;
    int64_t ts = std::max(t_move(bm * bn * out_b, s * r.epi_milli), t_move(cbytes, F * cal.hbm_milli));
    if (s > 1) ts += t_move((int64_t)(s - 1) * bm * bn * 4, s * cal.dsm_milli);
    const int64_t T = eq2(tl, trips, inner, ts);                      // Eq. 2
    int64_t cost;
    if (s == 1 && r.family != kSimt) {
        // persistent CTA + double-buffered TMEM (R11): Eq. 2 at the grid level
        cost = eq2(T - ts, F, ts, 0) + r.fixed;
    } else {
        cost = F * T + r.fixed + (s > 1 ? cal.fixed_cluster : 0);    // Eq. 4
    }
    o->rung_id = r.rung_id;
    o->split = s;
    o->family = r.family;
    o->swap = r.swap;
    o->bm = r.bm;
    o->bn = r.bn;
    o->stages = r.stages;
    o->tiles_m = (int32_t)tm;
    o->tiles_n = (int32_t)tn;
    o->grid = (int32_t)((s > 1 || r.family == kSimt) ? W : std::min(W, slots));
    o->cluster = (int32_t)(s * r.cg * mc);
    o->mc = (int32_t)mc;
    // R21: back to back, a first wave wider than half the SMs cannot become resident while
    // the previous grid holds its SMs (one full-SMEM CTA per SM)
    if (r.family != kSimt && std::min(W, slots) > d.sm_count / 2) cost += cal.stagger;
    o->cost = cost;
}

// Ragged batch (the varlen reading of BASELINE config 4): S_g = Q_g K_g^T
// for sequences of lengths s_g.  Eqs. 2-4 with the grid's aggregates: W = sum_g tiles_g
// (tiles cover each sequence separately: padding only at each sequence's edge), unique
// operand bytes in_b * K * 2 sum_g s_g, output bytes out_b * sum_g s_g^2; the persistent
// schedule's grid-level Eq. 2 (R11) and the stagger (R21) as for the uniform rungs.
static void varlen_cost(const vx_plan_s* p, const Rung& r, const int32_t* cu, int32_t ng,
                        vx_choice* o, int64_t* padded) {
    const vx_device_desc& d = p->desc;
    const Calib& cal = p->cal.glob;
    const int in_b = in_bytes(p->in), out_b = out_bytes(p->out);
    const int64_t bm = r.bm, bn = r.bn, bk = r.bk, K = p->K;
    int64_t tiles = 0, rows = 0, outs = 0, pad = 0;
    for (int32_t g = 0; g < ng; ++g) {
        const int64_t s = (int64_t)cu[g + 1] - cu[g];
        const int64_t tg = cdiv(s, bm) * cdiv(s, bn);
        tiles += tg;
        rows += s;
        outs += s * s;
        pad += cdiv(s, bm) * bm * cdiv(s, bn) * bn;
    }
    const int64_t kb = cdiv(K, bk);
    const int64_t slots = (int64_t)d.max_active_clusters[0];
    const int64_t W = std::max<int64_t>(tiles, 1);
    const int64_t F = eq3(W, slots);
    const int64_t inner = t_move(bm * bn * bk, r.mac_milli);
    const int64_t l_smem = t_move((bm + bn) * bk * in_b, r.l2s_milli);
    const int64_t l_hbm = t_move((int64_t)in_b * K * 2 * rows, F * kb * cal.hbm_milli);
    const int64_t tl = std::max(l_smem, l_hbm);
    const int64_t ts = std::max(t_move(bm * bn * out_b, r.epi_milli),
                                t_move((int64_t)out_b * outs, F * cal.hbm_milli));
    const int64_t T = eq2(tl, kb, inner, ts);
    int64_t cost = eq2(T - ts, F, ts, 0) + r.fixed;
    if (std::min(W, slots) > d.sm_count / 2) cost += cal.stagger;
    o->rung_id = r.rung_id; o->split = 1; o->family = r.family; o->swap = 0;
    o->bm = r.bm; o->bn = r.bn; o->stages = r.stages;
    o->tiles_m = 0; o->tiles_n = 0; o->grid = (int32_t)std::min(W, slots);
    o->cluster = 1; o->mc = 1;
    o->cost = cost;
    *padded = pad;
}

vx_status select_varlen(const vx_plan_s* p, const int32_t* cu, int32_t ng, int32_t force_rung,
                        vx_choice* out, int64_t* tiles) {
    bool have = false;
    vx_choice best{};
    int64_t best_pad = 0;
    for (const Rung& r : p->rungs) {
        // candidates: non-swapped cta_group::1 tcgen05 tiles, persistent (the varlen
        // epilogue stores each sequence's block from registers)
        if (r.family != kUmma || r.cg != 1 || r.mc != 1 || r.occ != 1) continue;
        if (force_rung >= 0 && r.rung_id != force_rung) continue;
        vx_choice c;
        int64_t pad = 0;
        varlen_cost(p, r, cu, ng, &c, &pad);
        if (!have || std::make_tuple(c.cost, pad, c.rung_id) < std::make_tuple(best.cost, best_pad, best.rung_id)) {
            best = c; best_pad = pad; have = true;
        }
    }
    if (!have) { set_error("rung %d cannot run a ragged batch", force_rung); return VX_ERR_INVALID; }
    int64_t t = 0;
    for (int32_t g = 0; g < ng; ++g) {
        const int64_t s = (int64_t)cu[g + 1] - cu[g];
        t += cdiv(s, best.bm) * cdiv(s, best.bn);
    }
    *tiles = t;
    *out = best;
    return VX_OK;
}

static inline int64_t padded_work(const vx_choice& c, int64_t batch) {
    // a multicast cluster pads its tile count to a multiple of mc along the non-shared axis
    const int64_t tm = (c.mc > 1 && c.swap) ? cdiv(c.tiles_m, c.mc) * c.mc : c.tiles_m;
    const int64_t tn = (c.mc > 1 && !c.swap) ? cdiv(c.tiles_n, c.mc) * c.mc : c.tiles_n;
    return batch * tm * c.bm * tn * c.bn;
}

static bool passes(int32_t filter, const Rung& r, int s) {
    if (filter == kSelectGather) return r.family == kUmma && (s == 0 || s == 1);
    return true;
}

vx_status select_choice(const vx_plan_s* p, int64_t batch, int64_t M, int64_t N,
                        int32_t force_rung, int32_t force_split, vx_choice* out,
                        int32_t filter) {
    if (!p || !out) { set_error("NULL argument"); return VX_ERR_INVALID; }
    if (batch < 1 || M < 1 || N < 1) { set_error("batch, M, N must be >= 1"); return VX_ERR_INVALID; }
    if (p->N > 0 && N != p->N) { set_error("N=%lld does not match the plan's N=%lld", (long long)N, (long long)p->N); return VX_ERR_INVALID; }
    if (force_rung >= 0) {
        if (force_rung >= (int32_t)p->rungs.size()) { set_error("rung %d not in table", force_rung); return VX_ERR_INVALID; }
        const Rung& r = p->rungs[force_rung];
        if (std::find(r.splits.begin(), r.splits.end(), force_split) == r.splits.end()) {
            set_error("split %d not admissible for rung %d", force_split, force_rung);
            return VX_ERR_INVALID;
        }
        if (r.family == kGemv && M > r.bm) {
            set_error("GEMV rung %d holds at most %d rows", force_rung, r.bm);
            return VX_ERR_INVALID;
        }
        if (!passes(filter, r, force_split)) {
            set_error("rung %d split %d cannot fan out rows (gather needs a non-swapped tcgen05 "
                      "rung with split 1 or 0)", force_rung, force_split);
            return VX_ERR_INVALID;
        }
        rung_cost(p, r, force_split, batch, M, N, out);
        return VX_OK;
    }
    const bool memo = batch == 1 && p->N > 0 && M <= vx_plan_s::kMemo && filter == kSelectAll;
    if (memo && p->memo_state[M].load(std::memory_order_acquire) == 2) {
        *out = p->memo[M];
        return VX_OK;
    }
    // Eq. 1 argmin, key (cost, padded work, rung_id, split) -- a total order (R13)
    bool have = false;
    vx_choice best{};
    for (const Rung& r : p->rungs)
        for (int s : r.splits) {
            if (s == 0 && !sk_admissible(p, r, batch, M, N)) continue;
            if (r.family == kGemv && M > r.bm) continue;   // GEMV rungs hold M <= MT rows
            if (!passes(filter, r, s)) continue;
            vx_choice c;
            rung_cost(p, r, s, batch, M, N, &c);
            if (!have || std::make_tuple(c.cost, padded_work(c, batch), c.rung_id, c.split) <
                             std::make_tuple(best.cost, padded_work(best, batch), best.rung_id, best.split)) {
                best = c;
                have = true;
            }
        }
    *out = best;
    if (memo) {
        uint8_t expect = 0;
        if (p->memo_state[M].compare_exchange_strong(expect, 1, std::memory_order_acq_rel)) {
            const_cast<vx_plan_s*>(p)->memo[M] = best;
            p->memo_state[M].store(2, std::memory_order_release);
        }
    }
    return VX_OK;
}

}  // namespace vx

using namespace vx;

static const char* dt_name(vx_dtype d) { return d == VX_BF16 ? "bf16" : d == VX_FP16 ? "fp16" : "fp32"; }

extern "C" {

int32_t vx_abi_version(void) { return VX_ABI_VERSION; }

const char* vx_status_str(vx_status s) {
    switch (s) {
    case VX_OK: return "VX_OK";
    case VX_ERR_INVALID: return "VX_ERR_INVALID";
    case VX_ERR_UNSUPPORTED: return "VX_ERR_UNSUPPORTED";
    case VX_ERR_ALIGN: return "VX_ERR_ALIGN";
    case VX_ERR_CUDA: return "VX_ERR_CUDA";
    case VX_ERR_NODEV: return "VX_ERR_NODEV";
    case VX_ERR_OOM: return "VX_ERR_OOM";
    case VX_ERR_BUFFER: return "VX_ERR_BUFFER";
    }
    return "VX_ERR_UNKNOWN";
}

const char* vx_last_error(void) { return g_err; }

static vx_status plan_create(int64_t N, int64_t K, vx_dtype in, vx_dtype out, vx_blayout bl,
                             const vx_device_desc* desc, const CalibTable& cal, vx_plan_t* plan) {
    g_err[0] = 0;
    if (!desc || !plan) { set_error("NULL argument"); return VX_ERR_INVALID; }
    *plan = nullptr;
    if (N < 0 || K <= 0) { set_error("need N >= 0 (0 = dynamic) and K > 0"); return VX_ERR_INVALID; }
    if ((int)in < 0 || (int)in > 2 || (int)out < 0 || (int)out > 2 || (int)bl < 0 || (int)bl > 2) {
        set_error("bad dtype or layout enum"); return VX_ERR_INVALID;
    }
    if (in == VX_FP32 && out != VX_FP32) { set_error("fp32 inputs need fp32 output"); return VX_ERR_UNSUPPORTED; }
    if (bl == VX_B_PACKED && (in == VX_FP32 || N == 0)) {
        set_error("VX_B_PACKED needs 16-bit inputs and a static N"); return VX_ERR_UNSUPPORTED;
    }
    if (in != VX_FP32 && (K % 8 != 0 || (bl == VX_B_KN && N > 0 && N % 8 != 0))) {
        set_error("16-bit inputs need K %% 8 == 0 (and N %% 8 == 0 when B is K x N): TMA 16-byte strides");
        return VX_ERR_ALIGN;
    }
    if (desc->sm_count <= 0 || desc->smem_optin <= 0 || desc->tmem_cols <= 0 ||
        desc->max_active_clusters[0] <= 0) {
        set_error("invalid device descriptor"); return VX_ERR_INVALID;
    }
    // resident clusters of size c can never exceed sm_count / c: the stream-K workspace has
    // sm_count slots and its flag spin-wait relies on every CTA of the grid being resident
    for (int i = 0; i < 4; ++i)
        if (desc->max_active_clusters[i] < 0 ||
            (int64_t)desc->max_active_clusters[i] * (1 << i) > desc->sm_count) {
            set_error("invalid device descriptor: max_active_clusters[%d]=%d exceeds sm_count/%d",
                      i, desc->max_active_clusters[i], 1 << i);
            return VX_ERR_INVALID;
        }
    std::unique_ptr<vx_plan_s> p(new (std::nothrow) vx_plan_s());
    if (!p) return VX_ERR_OOM;
    p->N = N; p->K = K; p->in = in; p->out = out; p->bl = bl; p->desc = *desc; p->device = -1;
    p->cal = cal;
    vx_status st = build_rungs(p.get());
    if (st != VX_OK) return st;
    p->memo.resize(vx_plan_s::kMemo + 1);
    p->memo_state.reset(new (std::nothrow) std::atomic<uint8_t>[vx_plan_s::kMemo + 1]);
    if (!p->memo_state) return VX_ERR_OOM;
    for (int64_t i = 0; i <= vx_plan_s::kMemo; ++i) p->memo_state[i].store(0);
    *plan = p.release();
    return VX_OK;
}

vx_status vx_plan_ex(int64_t N, int64_t K, vx_dtype in, vx_dtype out, vx_blayout bl,
                     const vx_device_desc* desc, vx_plan_t* plan) {
    return plan_create(N, K, in, out, bl, desc, builtin_calib(), plan);
}

vx_status vx_plan_ex_calibrated(int64_t N, int64_t K, vx_dtype in, vx_dtype out, vx_blayout bl,
                                const vx_device_desc* desc, vx_calib_t calib, vx_plan_t* plan) {
    if (!calib) { set_error("NULL calibration"); return VX_ERR_INVALID; }
    return plan_create(N, K, in, out, bl, desc, calib->table, plan);
}

vx_status vx_plan_calibrated(int64_t N, int64_t K, vx_dtype in, vx_dtype out, vx_blayout bl,
                             int device, vx_calib_t calib, vx_plan_t* plan) {
    if (!calib || !plan) { set_error("NULL argument"); return VX_ERR_INVALID; }
    vx_device_desc d;
    vx_status st = vx_device_probe(device, &d);
    if (st != VX_OK) return st;
    st = plan_create(N, K, in, out, bl, &d, calib->table, plan);
    if (st != VX_OK) return st;
    (*plan)->device = device;
    st = prepare_kernels(*plan);
    if (st != VX_OK) { vx_plan_destroy(*plan); *plan = nullptr; }
    return st;
}

vx_status vx_calib_new(int64_t hbm_milli, int64_t dsm_milli, int64_t fixed_cluster,
                       int64_t skfix_milli, int64_t stagger, vx_calib_t* out) {
    if (!out) { set_error("NULL argument"); return VX_ERR_INVALID; }
    if (hbm_milli <= 0 || dsm_milli <= 0 || fixed_cluster < 0 || skfix_milli <= 0 || stagger < 0) {
        set_error("calibration rates must be > 0"); return VX_ERR_INVALID;
    }
    vx_calib_s* c = new (std::nothrow) vx_calib_s();
    if (!c) return VX_ERR_OOM;
    c->table.glob = {hbm_milli, dsm_milli, fixed_cluster, skfix_milli, stagger};
    c->table.source = "user";
    *out = c;
    return VX_OK;
}

vx_status vx_calib_set_rung(vx_calib_t c, const char* key, int64_t mac_milli, int64_t l2s_milli,
                            int64_t epi_milli, int64_t fixed) {
    if (!c || !key) { set_error("NULL argument"); return VX_ERR_INVALID; }
    if (mac_milli <= 0 || l2s_milli <= 0 || epi_milli <= 0 || fixed < 0) {
        set_error("rung rates must be > 0"); return VX_ERR_INVALID;
    }
    for (auto& r : c->table.rungs)
        if (r.key == key) { r = {key, mac_milli, l2s_milli, epi_milli, fixed}; return VX_OK; }
    c->table.rungs.push_back({key, mac_milli, l2s_milli, epi_milli, fixed});
    return VX_OK;
}

vx_status vx_calib_destroy(vx_calib_t c) {
    delete c;
    return VX_OK;
}

vx_status vx_calib_dump(vx_calib_t c, char* buf, size_t cap, size_t* need) {
    const CalibTable& t = c ? c->table : builtin_calib();
    std::string s;
    char tmp[256];
    snprintf(tmp, sizeof tmp, "{\"source\":\"%s\",\"hbm_milli\":%lld,\"dsm_milli\":%lld,"
             "\"fixed_cluster\":%lld,\"skfix_milli\":%lld,\"stagger\":%lld,\"rungs\":{",
             t.source.c_str(), (long long)t.glob.hbm_milli, (long long)t.glob.dsm_milli,
             (long long)t.glob.fixed_cluster, (long long)t.glob.skfix_milli,
             (long long)t.glob.stagger);
    s += tmp;
    for (size_t i = 0; i < t.rungs.size(); ++i) {
        const RungConst& r = t.rungs[i];
        snprintf(tmp, sizeof tmp, "%s\"%s\":{\"mac_milli\":%lld,\"l2s_milli\":%lld,\"epi_milli\":%lld,"
                 "\"fixed\":%lld}", i ? "," : "", r.key.c_str(), (long long)r.mac_milli,
                 (long long)r.l2s_milli, (long long)r.epi_milli, (long long)r.fixed);
        s += tmp;
    }
    s += "}}";
    if (need) *need = s.size() + 1;
    if (!buf || cap < s.size() + 1) { set_error("dump buffer too small"); return VX_ERR_BUFFER; }
    memcpy(buf, s.c_str(), s.size() + 1);
    return VX_OK;
}

vx_status vx_plan(int64_t N, int64_t K, vx_dtype in, vx_dtype out, vx_blayout bl, int device,
                  vx_plan_t* plan) {
    vx_device_desc d;
    vx_status st = vx_device_probe(device, &d);
    if (st != VX_OK) return st;
    st = vx_plan_ex(N, K, in, out, bl, &d, plan);
    if (st != VX_OK) return st;
    (*plan)->device = device;
    st = prepare_kernels(*plan);
    if (st != VX_OK) { vx_plan_destroy(*plan); *plan = nullptr; }
    return st;
}

vx_status vx_plan_destroy(vx_plan_t plan) {
    delete plan;   // ~vx_plan_s releases the stream-K workspace (vx_dispatch.cu)
    return VX_OK;
}

vx_status vx_plan_select(vx_plan_t plan, int64_t batch, int64_t M, int64_t N, vx_choice* out) {
    return select_choice(plan, batch, M, N, -1, 0, out);
}

vx_status vx_plan_select_varlen(vx_plan_t plan, int32_t ngroups, const int32_t* cu,
                                vx_choice* out) {
    if (!plan || !cu || !out || ngroups < 1) { set_error("NULL argument or ngroups < 1"); return VX_ERR_INVALID; }
    for (int32_t g = 0; g < ngroups; ++g)
        if (cu[g + 1] < cu[g]) { set_error("cu_seqlens must be non-decreasing"); return VX_ERR_INVALID; }
    int64_t tiles = 0;
    return select_varlen(plan, cu, ngroups, -1, out, &tiles);
}

vx_status vx_plan_cost(vx_plan_t plan, int32_t rung_id, int32_t split, int64_t batch,
                       int64_t M, int64_t N, vx_choice* out) {
    if (rung_id < 0) { set_error("rung_id must be >= 0"); return VX_ERR_INVALID; }
    return select_choice(plan, batch, M, N, rung_id, split, out);
}

vx_status vx_plan_dump(vx_plan_t p, char* buf, size_t cap, size_t* need) {
    if (!p) { set_error("NULL plan"); return VX_ERR_INVALID; }
    std::string s;
    char tmp[512];
    const Calib& c = p->cal.glob;
    snprintf(tmp, sizeof tmp,
             "{\"abi\":%d,\"N\":%lld,\"K\":%lld,\"in\":\"%s\",\"out\":\"%s\",\"b_layout\":\"%s\","
             "\"levels\":{\"l0\":%lld,\"l1\":%lld,\"l2\":%lld,\"l3\":%lld},"
             "\"calib\":{\"hbm_milli\":%lld,\"dsm_milli\":%lld,\"fixed_cluster\":%lld,\"skfix_milli\":%lld,\"stagger\":%lld},\"rungs\":[",
             VX_ABI_VERSION, (long long)p->N, (long long)p->K, dt_name(p->in), dt_name(p->out),
             p->bl == VX_B_KN ? "kn" : p->bl == VX_B_NK ? "nk" : "packed", (long long)p->counts.l0, (long long)p->counts.l1,
             (long long)p->counts.l2, (long long)p->counts.l3, (long long)c.hbm_milli,
             (long long)c.dsm_milli, (long long)c.fixed_cluster, (long long)c.skfix_milli,
             (long long)c.stagger);
    s += tmp;
    for (size_t i = 0; i < p->rungs.size(); ++i) {
        const Rung& r = p->rungs[i];
        snprintf(tmp, sizeof tmp,
                 "%s{\"rung_id\":%d,\"family\":%d,\"cg\":%d,\"um\":%d,\"un\":%d,\"acc_stages\":%d,"
                 "\"bm\":%d,\"bn\":%d,\"bk\":%d,\"stages\":%d,\"swap\":%d,\"mc\":%d,\"occ\":%d,\"splits\":[",
                 i ? "," : "", r.rung_id, r.family, r.cg, r.um, r.un, r.acc_stages, r.bm, r.bn,
                 r.bk, r.stages, r.swap, r.mc, r.occ);
        s += tmp;
        for (size_t j = 0; j < r.splits.size(); ++j) {
            snprintf(tmp, sizeof tmp, "%s%d", j ? "," : "", r.splits[j]);
            s += tmp;
        }
        snprintf(tmp, sizeof tmp, "],\"mac_milli\":%lld,\"l2s_milli\":%lld,\"epi_milli\":%lld,\"fixed\":%lld}",
                 (long long)r.mac_milli, (long long)r.l2s_milli, (long long)r.epi_milli, (long long)r.fixed);
        s += tmp;
    }
    s += "]}";
    if (need) *need = s.size() + 1;
    if (!buf || cap < s.size() + 1) { set_error("dump buffer too small"); return VX_ERR_BUFFER; }
    memcpy(buf, s.c_str(), s.size() + 1);
    return VX_OK;
}

}  // extern "C"
