// C ABI of libtmotif (include/tmotif.h): argument validation, motif
// canonicalisation, the per-query horizon construction and the mining
// launch.  Every step of the hot path runs in this library's kernels.
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "catalog.cuh"


namespace tmg {

tm_status graph_create(const uint32_t *src, const uint32_t *dst, const int64_t *t, uint64_t m, uint32_t n,
                       const tm_graph_opts *o, tm_graph **out);
void graph_destroy(tm_graph *g);
cudaError_t build_horizons(const DeviceGraph &d, int64_t d0, int64_t d1, uint32_t *H0, uint32_t *H1, cudaStream_t s);
cudaError_t build_hrank(const DeviceGraph &d, int var, const uint32_t *H, uint32_t *R, cudaStream_t s,
                        uint4 *W = nullptr);
cudaError_t build_tie_lo(const DeviceGraph &d, uint32_t *S, cudaStream_t s);
tm_status set_labels(DeviceGraph &d, const int32_t *vl, const int32_t *el, bool on_device);

namespace {
thread_local std::string g_err;
thread_local tm_run_info g_info = {};

std::vector<CatalogEntry> &catalog() {
    static std::vector<CatalogEntry> v = [] {
        std::vector<CatalogEntry> c;
        register_named(c);
        register_p36_part<0>(c);
        register_p36_part<1>(c);
        register_p36_part<2>(c);
        register_p36_part<3>(c);
        return c;
    }();
    return v;
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (dev >= 0 && dev != prev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

std::mutex g_attr_mu;
std::unordered_map<const void *, int> g_attr_done;  // kernel -> dynamic smem configured

}  // namespace

void set_error(const std::string &msg) { g_err = msg; }
tm_status fail(tm_status st, const std::string &msg) {
    g_err = msg;
    return st;
}

bool is_specialised(uint64_t code) {
    for (auto &e : catalog())
        if (e.code == code) return true;
    return false;
}

KernelInfo lookup_kernel(uint64_t code, int mode, bool *specialised, bool generic) {
    if (!generic && (mode == kCount || mode == kEnum || mode == kCountPfx || mode == kResume || mode == kCountSib)) {
        for (auto &e : catalog()) {
            if (e.code != code) continue;
            const KernelInfo &ki = mode == kCount ? e.count : mode == kEnum ? e.enumerate
                                 : mode == kCountPfx ? e.count_pfx : mode == kResume ? e.resume : e.count_sib;
            if (!ki.fn) break;
            if (specialised) *specialised = true;
            return ki;
        }
    }
    if (specialised) *specialised = false;
    switch (mode) {
        case kCount: return kernel_info<PlanR, kCount>();
        case kCountPfx: return kernel_info<PlanR, kCountPfx>();
        case kResume: return kernel_info<PlanR, kResume>();
        case kCountSib: return kernel_info<PlanR, kCountSib>();
        case kEnum: return kernel_info<PlanR, kEnum>();
        case kRoots: return kernel_info<PlanR, kRoots>();
        default: return kernel_info<PlanR, kStats>();
    }
}

namespace {

struct RunOut {
    uint64_t count = 0;
    uint64_t stats[kScratchWords] = {};
};

// One query over k motifs (k = 1: tm_count & co; k > 1: tm_count_multi):
// the δ-horizons of every distinct δ / δ_i and the window-end ranks of every
// distinct (list variant, gap horizon) are built once, then one mining kernel
// per motif runs on the same stream.
thread_local std::vector<tm_kernel_info> g_kinfo;
static_assert(TM_KMODE_COUNT == kCount && TM_KMODE_ENUM == kEnum && TM_KMODE_COUNT_PREFIX == kCountPfx &&
                  TM_KMODE_RESUME == kResume && TM_KMODE_COUNT_SIB == kCountSib,
              "tmotif.h kernel modes follow tmg::Mode");

tm_status run_multi(const tm_graph *g, const tm_motif *const *mos, uint32_t k, const tm_run_opts *opts, int mode,
                    uint32_t *enum_dev, uint64_t cap, const uint64_t *roots_dev, uint64_t n_roots_list,
                    unsigned long long *root_counts_dev, RunOut *out) {
    if (!g || !mos || k == 0) return fail(TM_EINVAL, "null graph or motif");
    for (uint32_t i = 0; i < k; i++) {
        if (!mos[i]) return fail(TM_EINVAL, "null motif");
        if (mos[i]->disconnected && (mos[i]->constrained() || mode == kStats))
            return fail(TM_EUNSUPPORTED, "prefix-disconnected motifs (Q9) support count / enumerate / per-root "
                                         "counts without labels or anti-edges");
    }
    tm_run_opts o;
    tm_run_opts_default(&o);
    if (opts) o = *opts;
    if (o.share < 0 || o.share > 2) return fail(TM_EINVAL, "tm_run_opts.share must be 0, 1 or 2");
    DeviceGuard guard(g->device);
    cudaStream_t s = (cudaStream_t)o.stream;
    const DeviceGraph &d = g->d;
    const uint64_t m = d.m;
    g_info = tm_run_info{};
    {
        tm_kernel_info none{};
        none.carried_by = -1;
        none.kernel_mode = TM_KMODE_NONE;
        g_kinfo.assign(k, none);
    }
    if (o.edge_id_offset + m > (1ull << 32)) return fail(TM_EINVAL, "edge_id_offset + m exceeds 2^32");

    MineParams base;
    std::memset(&base, 0, sizeof base);
    base.src = d.src; base.dst = d.dst; base.off_out = d.off_out; base.off_in = d.off_in; base.rec = d.rec;
    base.rank = d.rank;
    base.m = (uint32_t)m;
    base.split = (uint32_t)(m + d.n);
    base.prec = d.prec; base.ptab = d.ptab; base.pmask = d.pmask; base.pbits = d.pbits; base.fmask = d.fmask;
    base.tbits = d.tbits; base.tmask = d.tmask; base.tshift = d.tshift;
    if (roots_dev) {
        base.roots = roots_dev;
        base.n_roots = n_roots_list;
    } else {
        uint64_t hi = std::min<uint64_t>(o.root_hi, m), lo = std::min<uint64_t>(o.root_lo, hi);
        base.root_lo = lo;
        base.n_roots = hi - lo;
    }
    base.id_offset = (uint32_t)o.edge_id_offset;
    base.enum_buf = enum_dev;
    base.cap = cap;
    base.root_counts = root_counts_dev;
    base.share = o.share;

    // distinct horizons over all motifs: each δ, and every finite δ_i < δ (a
    // gap bound >= δ can never bind: t_prev >= t_root)
    std::vector<int64_t> hv;
    auto hidx = [&](int64_t x) {
        auto it = std::find(hv.begin(), hv.end(), x);
        if (it != hv.end()) return (int)(it - hv.begin());
        hv.push_back(x);
        return (int)hv.size() - 1;
    };
    std::vector<int> dl(k, -1);
    std::vector<std::array<int, kMaxL>> gap(k);
    std::vector<std::pair<int, int>> hkeys;   // window-end ranks: (list variant, horizon index)
    std::vector<std::array<int, kMaxL>> hwhich(k);
    std::vector<std::array<int, TM_MAX_ANTI>> anti_h(k);   // horizon index of each anti-edge window
    bool need_tie = false;                                 // tie_lo: first id of each timestamp
    for (uint32_t i = 0; i < k; i++) {
        const tm_motif *mo = mos[i];
        gap[i].fill(-1);
        hwhich[i].fill(-1);
        anti_h[i].fill(-1);
        if ((mo->L < 2 && !mo->n_anti) || base.n_roots == 0) continue;
        dl[i] = hidx(mo->delta);
        for (uint32_t j = 0; j < mo->n_anti; j++) anti_h[i][j] = hidx(mo->anti_window[j]);
        if (mo->n_anti) need_tie = true;
        for (uint32_t j = 0; j + 1 < mo->L; j++) {
            const int64_t f = mo->fine[j];
            if (f == TM_DELTA_INF || f >= mo->delta) continue;
            gap[i][j] = hidx(f);
        }
        // window-end ranks (build_hrank) for the levels whose list is anchored at
        // the previous edge and bounded by a gap horizon.  The instrumentation
        // run (kStats) does not use them.
        if (!TM_HRANK || mode == kStats || mo->disconnected) continue;
        Shape sh{};
        sh.L = (int)mo->L;
        for (uint32_t j = 0; j < mo->L; j++) { sh.u[j] = mo->u[j]; sh.v[j] = mo->v[j]; }
        for (int nl = 1; nl < sh.L; nl++) {
            if (gap[i][nl - 1] < 0 || sh.pairk(nl) || sh.anc(nl) != nl - 1) continue;
            const std::pair<int, int> key{sh.avar(nl), gap[i][nl - 1]};
            auto it = std::find(hkeys.begin(), hkeys.end(), key);
            hwhich[i][nl - 1] = (int)(it - hkeys.begin());
            if (it == hkeys.end()) hkeys.push_back(key);
        }
    }

    // sibling emission + resume: motif B = A's first K edges + one closing edge
    // whose candidates are A's level-K candidates (same list, same window), A
    // continuing past level K+1: A's kernel writes B's matches as rows; B's
    // count is their number, and a motif D that starts with B continues from
    // those rows at level K+1 (a kResume kernel) instead of searching again
    std::vector<int> sib_of(k, -1), resume_of(k, -1);
    std::vector<uint32_t> sib_vtx(k, 0), sib_K(k, 0);
    if (mode == kCount && o.fuse == 0 && k > 1) {
        auto eff = [](const tm_motif *mo, uint32_t g) {
            const int64_t f = mo->fine[g];
            return (f == TM_DELTA_INF || f >= mo->delta) ? TM_DELTA_INF : f;
        };
        auto shape = [](const tm_motif *mo) {
            Shape sh{};
            sh.L = (int)mo->L;
            for (uint32_t j = 0; j < mo->L; j++) { sh.u[j] = mo->u[j]; sh.v[j] = mo->v[j]; }
            return sh;
        };
        auto plain = [](const tm_motif *mo) {
            return !mo->constrained() && !mo->rtc_fn[kCount] && !mo->disconnected;
        };
        for (uint32_t b = 0; b < k; b++) {   // B: a sibling of a launched motif A
            const tm_motif *mb = mos[b];
            if (!plain(mb) || mb->L < 2) continue;
            const uint32_t K = mb->L - 1;
            if (K != (uint32_t)kSibLevel) continue;   // the kCountSib kernels emit at level 2
            const Shape sb = shape(mb);
            const int nbk = sb.nv((int)K);
            if (!(sb.u[K] < nbk && sb.v[K] < nbk)) continue;   // B's last edge must close (both ends mapped)
            for (uint32_t a = 0; a < k && sib_of[b] < 0; a++) {
                const tm_motif *ma = mos[a];
                if (a == b || sib_of[a] >= 0 || !plain(ma) || ma->L < K + 2 ||
                    ma->delta != mb->delta)
                    continue;
                if (motif_code((int)K, ma->u, ma->v) != motif_code((int)K, mb->u, mb->v)) continue;
                bool same = true;
                for (uint32_t g = 0; g < K; g++) same &= eff(ma, g) == eff(mb, g);
                if (!same) continue;
                const Shape sa = shape(ma);
                const int nak = sa.nv((int)K);
                if (sa.u[K] < nak && sa.v[K] < nak) continue;        // A's edge K must be open (full windows)
                if (sa.ldir((int)K) != sb.ldir((int)K) || sa.lx((int)K) != sb.lx((int)K)) continue;
                sib_of[b] = (int)a;
                sib_K[b] = K;
                sib_vtx[b] = (uint32_t)(sb.ldir((int)K) == 0 ? sb.v[K] : sb.u[K]);
            }
        }
        for (uint32_t d = 0; d < k; d++) {   // D: continues from the rows of a sibling B
            const tm_motif *md = mos[d];
            if (sib_of[d] >= 0 || !plain(md)) continue;
            for (uint32_t b = 0; b < k && resume_of[d] < 0; b++) {
                const tm_motif *mb = mos[b];
                if (sib_of[b] < 0 || (int)d == sib_of[b] || md->L <= mb->L || md->delta != mb->delta) continue;
                if (motif_code((int)mb->L, md->u, md->v) != mb->code) continue;
                bool same = true;
                for (uint32_t g = 0; g + 1 < mb->L; g++) same &= eff(md, g) == eff(mb, g);
                if (same) resume_of[d] = (int)b;
            }
        }
    }
    // at most one sibling per carrier kernel
    {
        std::vector<int> taken(k, 0);
        for (uint32_t b = 0; b < k; b++)
            if (sib_of[b] >= 0) {
                if (taken[sib_of[b]]) sib_of[b] = -1;
                else taken[sib_of[b]] = 1;
            }
        for (uint32_t d = 0; d < k; d++)
            if (resume_of[d] >= 0 && sib_of[resume_of[d]] < 0) resume_of[d] = -1;
    }
    // a carrier of a sibling runs in the kCountPfx mode; prefix fusion of the
    // sibling's own prefixes is unaffected
    // prefix fusion (counting): the longest motifs run their kernels; a motif
    // that is the first l edges of one of them, with the same δ and effective
    // δ_1..δ_{l-1} and no constraints, is counted there as its level-l nodes
    std::vector<int> carrier(k, -1);
    std::vector<uint32_t> pmask(k, 0);
    if (mode == kCount && o.fuse == 0 && k > 1) {
        std::vector<uint32_t> order(k);
        for (uint32_t i = 0; i < k; i++) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return mos[a]->L > mos[b]->L; });
        auto eff = [](const tm_motif *mo, uint32_t g) {
            const int64_t f = mo->fine[g];
            return (f == TM_DELTA_INF || f >= mo->delta) ? TM_DELTA_INF : f;
        };
        // a motif whose kernel writes a sibling's rows (sib_of[b] == i) must run
        // that kernel: handing it to a longer carrier would leave the sibling
        // (and whatever resumes from its rows) at 0
        std::vector<char> sib_carrier(k, 0);
        for (uint32_t b = 0; b < k; b++)
            if (sib_of[b] >= 0) sib_carrier[sib_of[b]] = 1;
        for (uint32_t a = 0; a < k; a++) {
            const uint32_t i = order[a];
            const tm_motif *mi = mos[i];
            if (mi->constrained() || mi->disconnected || sib_of[i] >= 0 || resume_of[i] >= 0 || sib_carrier[i])
                continue;
            for (uint32_t b = 0; b < a && carrier[i] < 0; b++) {
                const uint32_t j = order[b];
                const tm_motif *mj = mos[j];
                if (carrier[j] >= 0 || sib_of[j] >= 0 || resume_of[j] >= 0 || mj->constrained() || mj->disconnected ||
                    mj->rtc_fn[kCount] || mj->L <= mi->L ||
                    mj->delta != mi->delta)
                    continue;
                if (motif_code((int)mi->L, mj->u, mj->v) != mi->code) continue;
                bool same = true;
                for (uint32_t g = 0; g + 1 < mi->L; g++) same &= eff(mi, g) == eff(mj, g);
                if (!same) continue;
                carrier[i] = (int)j;
                pmask[j] |= 1u << mi->L;
            }
        }
    }

    uint32_t *sib_rows = nullptr;
    uint64_t sib_cap = 0;

    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evd = nullptr;
    std::vector<cudaEvent_t> evk(k, nullptr);
    struct EvFree {
        std::vector<cudaEvent_t *> e;
        ~EvFree() { for (auto *p : e) if (*p) cudaEventDestroy(*p); }
    } evf;
    for (cudaEvent_t *e : {&ev0, &ev1, &evd}) { TM_CUDA_TRY(cudaEventCreate(e)); evf.e.push_back(e); }
    for (auto &e : evk) { TM_CUDA_TRY(cudaEventCreate(&e)); evf.e.push_back(&e); }

    struct Free {
        std::vector<void *> v;
        cudaStream_t s;
        ~Free() { for (void *p : v) dev_free(p, s); }
    } fr{{}, s};
    unsigned long long *scratch = nullptr;
    TM_CUDA_TRY(dev_alloc((void **)&scratch, (size_t)k * kScratchWords * sizeof(unsigned long long), s));
    fr.v.push_back(scratch);
    TM_CUDA_TRY(cudaMemsetAsync(scratch, 0, (size_t)k * kScratchWords * sizeof(unsigned long long), s));
    uint32_t *hbuf = nullptr, *hrbuf = nullptr;
    const uint64_t mh = (m + 3) & ~3ull;   // horizon stride: 16-byte aligned arrays (vector stores)
    if (!hv.empty()) {
        TM_CUDA_TRY(dev_alloc((void **)&hbuf, hv.size() * mh * sizeof(uint32_t), s));
        fr.v.push_back(hbuf);
    }
    const size_t hr_elem = TM_HRANK == 3 ? sizeof(uint4) : sizeof(uint32_t);
    if (!hkeys.empty()) {
        TM_CUDA_TRY(dev_alloc((void **)&hrbuf, hkeys.size() * m * hr_elem, s));
        fr.v.push_back(hrbuf);
    }
    uint32_t *tie = nullptr;
    if (need_tie && m) {
        TM_CUDA_TRY(dev_alloc((void **)&tie, m * sizeof(uint32_t), s));
        fr.v.push_back(tie);
    }

    TM_CUDA_TRY(cudaEventRecord(ev0, s));
    NvtxRange nv_passes("tm.query_passes (horizons, window descriptors)");
    for (size_t i = 0; i < hv.size(); i += 2) {   // two horizons per pass (one read of T)
        const bool two = i + 1 < hv.size();
        TM_CUDA_TRY(build_horizons(d, hv[i], two ? hv[i + 1] : hv[i], hbuf + i * mh, two ? hbuf + (i + 1) * mh : nullptr, s));
        g_info.launches += 2;
    }
    if (tie) {
        TM_CUDA_TRY(build_tie_lo(d, tie, s));
        g_info.launches++;
    }
    if (!hkeys.empty()) {
        if (TM_HRANK == 2) {   // memo: 0 = not yet known
            TM_CUDA_TRY(cudaMemsetAsync(hrbuf, 0, hkeys.size() * m * sizeof(uint32_t), s));
        } else {
            for (size_t i = 0; i < hkeys.size(); i++) {
                uint32_t *Hh = hbuf + (size_t)hkeys[i].second * mh;
                if (TM_HRANK == 3) {
                    TM_CUDA_TRY(build_hrank(d, hkeys[i].first, Hh, nullptr, s, (uint4 *)hrbuf + i * m));
                } else {
                    TM_CUDA_TRY(build_hrank(d, hkeys[i].first, Hh, hrbuf + i * m, s));
                }
                g_info.launches++;
            }
        }
    }
    TM_CUDA_TRY(cudaEventRecord(ev1, s));

    void *qbuf = nullptr;   // heavy-subtree sharing queue, reused by the launches (stream order)
    uint32_t qcap = 0;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    TM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int threads = kWarpsPerBlock * 32;
    // sibling rows: one region per sibling motif (cap rows of L_b edge ids)
    // (a sibling nobody resumes from is only counted: no rows, cap 0)
    std::vector<uint32_t *> sib_region(k, nullptr);
    std::vector<char> rows_needed(k, 0);
    for (uint32_t d = 0; d < k; d++)
        if (resume_of[d] >= 0) rows_needed[resume_of[d]] = 1;
    {
        uint64_t words = 0;
        sib_cap = std::min<uint64_t>(std::max<uint64_t>(base.n_roots, 1u << 16), 1u << 22);
        for (uint32_t b = 0; b < k; b++)
            if (sib_of[b] >= 0 && rows_needed[b]) words += sib_cap * mos[b]->L;
        if (words) {
            TM_CUDA_TRY(dev_alloc((void **)&sib_rows, words * sizeof(uint32_t), s));
            fr.v.push_back(sib_rows);
            uint64_t off = 0;
            for (uint32_t b = 0; b < k; b++)
                if (sib_of[b] >= 0 && rows_needed[b]) {
                    sib_region[b] = sib_rows + off;
                    off += sib_cap * mos[b]->L;
                }
        }
    }
    // launch order: every searching kernel, then the kernels resuming from sibling rows
    std::vector<uint32_t> ord;
    for (uint32_t i = 0; i < k; i++)
        if (resume_of[i] < 0) ord.push_back(i);
    for (uint32_t i = 0; i < k; i++)
        if (resume_of[i] >= 0) ord.push_back(i);
    std::vector<int> pos_of(k, 0);
    for (uint32_t oi = 0; oi < k; oi++) pos_of[ord[oi]] = (int)oi;
    for (uint32_t oi = 0; oi < k; oi++) {
        const uint32_t i = ord[oi];
        const tm_motif *mo = mos[i];
        if (carrier[i] >= 0 || sib_of[i] >= 0) {   // counted inside another motif's kernel
            TM_CUDA_TRY(cudaEventRecord(evk[i], s));
            continue;
        }
        NvtxRange nv_mine(resume_of[i] >= 0 ? "tm.mine (resume)" : "tm.mine");
        MineParams p = base;
        p.prefix_mask = pmask[i];
        p.prefix_lv0 = pmask[i] ? (uint32_t)__builtin_ctz(pmask[i]) : 0u;
        for (uint32_t b = 0; b < k; b++)
            if (sib_of[b] == (int)i) {   // this kernel emits sibling b's matches as rows
                p.sib_level = sib_K[b];
                p.sib_vtx = sib_vtx[b];
                p.sib_rows = sib_region[b];
                p.sib_cap = rows_needed[b] ? (uint32_t)sib_cap : 0u;
            }
        // root pruning (TM_ROOT_PRUNE): every match of this motif closes with an edge
        // in the root endpoint y's list inside (e_1, H_δ(e_1)] (the closing
        // look-ahead window); when that window is empty the root has no
        // match.  Only when no node count is needed (no prefix counting) and a
        // sibling emitted by this kernel, if any, closes through the same list.
        p.root_prune = 0;
        if (TM_ROOT_PRUNE && (mode == kCount || mode == kEnum || mode == kRoots) && !mo->constrained() &&
            !mo->disconnected && pmask[i] == 0) {
            Shape sh{};
            sh.L = (int)mo->L;
            for (uint32_t j = 0; j < mo->L; j++) { sh.u[j] = mo->u[j]; sh.v[j] = mo->v[j]; }
            bool ok = sh.look();
            for (uint32_t b = 0; b < k && ok; b++)
                if (sib_of[b] == (int)i) {
                    const tm_motif *mb = mos[b];
                    const uint32_t K = mb->L - 1;
                    const int y = sh.lky();
                    ok = sh.lkdir() == 1 ? ((int)mb->v[K] == y && (int)mb->u[K] != y)
                                         : ((int)mb->u[K] == y && (int)mb->v[K] != y);
                }
            p.root_prune = ok ? 1u : 0u;
        }
        const bool resuming = resume_of[i] >= 0;
        if (resuming) {   // continue from sibling b's rows
            const int b = resume_of[i];
            p.resume_rows = sib_region[b];
            p.resume_n = scratch + (size_t)sib_of[b] * kScratchWords + kSibCount;
            p.resume_level = mos[b]->L;
            p.sib_cap = (uint32_t)sib_cap;
            p.roots = nullptr;
            p.root_lo = 0;
            p.n_roots = sib_cap;   // grid sizing; the kernel reads the row count
        }
        p.L = mo->L;
        for (uint32_t j = 0; j < mo->L; j++) { p.u[j] = mo->u[j]; p.v[j] = mo->v[j]; }
        p.scratch = scratch + (size_t)i * kScratchWords;
        if (mo->constrained()) {   // generalized query: the generic kernel checks labels and anti-edges
            p.gen = 1;
            p.vlab = d.vlab;
            p.elab = d.elab;
            for (int j = 0; j < kMaxV; j++) p.vreq[j] = mo->vreq[j];
            for (int j = 0; j < kMaxL; j++) p.ereq[j] = mo->ereq[j];
            p.n_anti = mo->n_anti;
            for (uint32_t j = 0; j < mo->n_anti; j++) {
                p.anti_u[j] = mo->anti_u[j];
                p.anti_v[j] = mo->anti_v[j];
                p.anti_a[j] = mo->anti_attach[j];
                p.anti_hi[j] = dl[i] >= 0 ? hbuf + (size_t)anti_h[i][j] * mh : nullptr;
            }
            p.tie_lo = tie;
        }
        if (dl[i] >= 0) {
            p.H = hbuf + (size_t)dl[i] * mh;
            for (uint32_t j = 0; j + 1 < mo->L; j++) {
                p.Hf[j] = gap[i][j] >= 0 ? hbuf + (size_t)gap[i][j] * mh : nullptr;
                if (TM_HRANK == 3)
                    p.HW[j] = hwhich[i][j] >= 0 ? (const uint4 *)hrbuf + (size_t)hwhich[i][j] * m : nullptr;
                else
                    p.HR[j] = hwhich[i][j] >= 0 ? hrbuf + (size_t)hwhich[i][j] * m : nullptr;
            }
        }
        if (p.n_roots > 0 && mo->disconnected) {   // two new vertices at one level: dfs.cu
            uint32_t grid = 0;
            TM_CUDA_TRY(launch_mine_dfs(p, mode, sms, s, &grid));
            g_info.launches++;
            g_info.grid_ctas = grid;
            g_info.block_threads = 256;
            g_kinfo[i].grid_ctas = grid;
            g_kinfo[i].kernel_mode = TM_KMODE_DFS;
        } else if (p.n_roots > 0) {
            bool spec = false;
            // a runtime-specialised kernel (tm_motif_specialise) first, then the
            // build-time catalog, then the generic kernel
            const int kmode = resuming ? (int)kResume
                              : (mode == kCount && p.sib_level) ? (int)kCountSib
                              : (mode == kCount && p.prefix_mask) ? (int)kCountPfx : mode;
            void *rfn = (kmode == kCount || kmode == kEnum) ? mo->rtc_fn[kmode] : nullptr;
            KernelInfo ki{nullptr, 0};
            if (!rfn) ki = lookup_kernel(mo->code, kmode, &spec, mo->constrained());
            const size_t smem = (size_t)(rfn ? mo->rtc_smem[mode] : ki.smem_per_warp) * kWarpsPerBlock;
            {
                std::lock_guard<std::mutex> lk(g_attr_mu);
                auto key = rfn ? (const void *)rfn : (const void *)ki.fn;
                if (!g_attr_done.count(key)) {
                    if (rfn) {
                        TM_CUDA_TRY(rtc_set_smem(rfn, (int)smem));
                    } else {
                        TM_CUDA_TRY(cudaFuncSetAttribute(ki.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         (int)smem));
#ifdef TM_CARVEOUT_MAX
                        TM_CUDA_TRY(cudaFuncSetAttribute(ki.fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                                         (int)cudaSharedmemCarveoutMaxShared));
#endif
                    }
                    g_attr_done[key] = 1;
                }
            }
            int per_sm = 0;
            if (rfn) {
                TM_CUDA_TRY(rtc_occupancy(rfn, threads, smem, &per_sm));
            } else {
                TM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ki.fn, threads, smem));
            }
            if (per_sm < 1) return fail(TM_ECUDA, "mining kernel does not fit on an SM");
            uint64_t grid = o.grid_ctas ? o.grid_ctas : (uint64_t)sms * per_sm;
            // no more warps than 32-root batches
            uint64_t max_useful = (p.n_roots + 31) / 32;
            max_useful = (max_useful + kWarpsPerBlock - 1) / kWarpsPerBlock;
            grid = std::max<uint64_t>(1, std::min(grid, max_useful));
            // heavy-subtree sharing: idle warps wait for work, so every CTA must
            // be resident at once (a CTA waiting for a slot would never start):
            // the grid is capped at the co-resident limit and launched
            // cooperatively, which the driver either schedules all at once or
            // refuses (cudaErrorCooperativeLaunchTooLarge) — two sharing kernels
            // on different streams can then never each hold part of the GPU
            // while waiting for the rest
            const bool coop = p.share != 1;
            if (coop) {
                grid = std::min<uint64_t>(grid, (uint64_t)sms * per_sm);
                p.total_warps = (uint32_t)(grid * kWarpsPerBlock);
                uint32_t q = 32;
                while (q < p.total_warps) q <<= 1;
                if (q > qcap) {
                    if (qbuf) dev_free(qbuf, s);
                    qbuf = nullptr;
                    TM_CUDA_TRY(dev_alloc(&qbuf, (size_t)q * (sizeof(unsigned) + kShareWords * sizeof(uint32_t)), s));
                    qcap = q;
                }
                p.qmask = q - 1;
                p.qflag = (unsigned *)qbuf;
                p.qrec = (uint32_t *)((char *)qbuf + (size_t)q * sizeof(unsigned));
                TM_CUDA_TRY(cudaMemsetAsync(p.qflag, 0, (size_t)q * sizeof(unsigned), s));
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)grid);
            cfg.blockDim = dim3(threads);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeCooperative;
            attr[0].val.cooperative = 1;
            cfg.attrs = attr;
            cfg.numAttrs = coop ? 1 : 0;
            if (rfn) {
                TM_CUDA_TRY(rtc_launch(rfn, (unsigned)grid, threads, smem, s, p, coop));
            } else {
                TM_CUDA_TRY(cudaLaunchKernelEx(&cfg, ki.fn, p));
            }
            g_info.launches++;
            g_info.grid_ctas = (uint32_t)grid;
            g_info.block_threads = threads;
            g_kinfo[i].grid_ctas = (uint32_t)grid;
            g_kinfo[i].kernel_mode = kmode;
        }
        TM_CUDA_TRY(cudaEventRecord(evk[i], s));
    }
    if (qbuf) fr.v.push_back(qbuf);
    std::vector<unsigned long long> host((size_t)k * kScratchWords);
    TM_CUDA_TRY(cudaMemcpyAsync(host.data(), scratch, host.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                s));
    TM_CUDA_TRY(cudaEventRecord(evd, s));
    TM_CUDA_TRY(cudaStreamSynchronize(s));
    cudaEventElapsedTime(&g_info.horizon_ms, ev0, ev1);
    cudaEventElapsedTime(&g_info.mine_ms, ev1, evk[ord.back()]);
    cudaEventElapsedTime(&g_info.total_ms, ev0, evd);
    for (uint32_t i = 0; i < k; i++) {
        const unsigned long long *h = host.data() + (size_t)i * kScratchWords;
        tm_kernel_info &ki = g_kinfo[i];
        cudaEventElapsedTime(&ki.mine_ms, pos_of[i] ? evk[ord[pos_of[i] - 1]] : ev1, evk[i]);
        ki.shared_tasks = h[kShareDone];
        if (h[kTimeStart] && h[kTimeExit]) {
            const unsigned long long t0 = ~h[kTimeStart], te = h[kTimeExit];
            const unsigned long long td = h[kTimeDrain] ? ~h[kTimeDrain] : te;
            ki.tail_ms = te > td ? (float)((te - td) * 1e-6) : 0.f;
            if (te > t0 && ki.grid_ctas)
                ki.warp_busy = (float)(((double)h[kTimeBusy] - (double)h[kTimeWait]) /
                                       ((double)(te - t0) * ki.grid_ctas * kWarpsPerBlock));
        }
        out[i].count = mode == kEnum ? h[2] : h[1];
        ki.carried_by = carrier[i];
        if (carrier[i] >= 0) {
            out[i].count = host[(size_t)carrier[i] * kScratchWords + kPrefixBase + mos[i]->L];
            ki = tm_kernel_info{};
            ki.carried_by = carrier[i];
            ki.kernel_mode = TM_KMODE_NONE;
        } else if (sib_of[i] >= 0) {   // sibling: the number of rows its carrier emitted
            out[i].count = host[(size_t)sib_of[i] * kScratchWords + kSibCount];
            ki = tm_kernel_info{};
            ki.carried_by = sib_of[i];
            ki.kernel_mode = TM_KMODE_NONE;
        }
        for (int w = 0; w < kScratchWords; w++) out[i].stats[w] = h[w];
#ifdef TM_PHASE_PROFILE
        fprintf(stderr, "[phase]");
        for (int l = 0; l < 6; l++)
            if (h[21 + 2 * l])
                fprintf(stderr, " L%d: steps=%llu cyc/step=%.0f share=%.3f", l, h[21 + 2 * l],
                        (double)h[20 + 2 * l] / h[21 + 2 * l], 0.0 + h[20 + 2 * l]);
        fprintf(stderr, "\n");
#endif
    }
    // a sibling with more matches than row slots: its resuming motifs are
    // counted again from scratch (without fusion)
    for (uint32_t d = 0; d < k; d++) {
        if (resume_of[d] < 0) continue;
        const int b = resume_of[d];
        if (host[(size_t)sib_of[b] * kScratchWords + kSibCount] <= sib_cap) continue;
        const std::vector<tm_kernel_info> keep = g_kinfo;
        const tm_run_info keep_info = g_info;
        tm_run_opts o2 = o;
        o2.fuse = 1;
        RunOut r2;
        const tm_status st = run_multi(g, &mos[d], 1, &o2, mode, nullptr, 0, nullptr, 0, nullptr, &r2);
        g_kinfo = keep;
        g_info = keep_info;
        if (st) return st;
        out[d].count = r2.count;
    }
    // the last motif's load balance in the single-query record
    g_info.shared_tasks = g_kinfo[k - 1].shared_tasks;
    g_info.tail_ms = g_kinfo[k - 1].tail_ms;
    g_info.warp_busy = g_kinfo[k - 1].warp_busy;
    return TM_OK;
}

tm_status run(const tm_graph *g, const tm_motif *mo, const tm_run_opts *opts, int mode, uint32_t *enum_dev,
              uint64_t cap, const uint64_t *roots_dev, uint64_t n_roots_list, unsigned long long *root_counts_dev,
              RunOut *out) {
    return run_multi(g, &mo, 1, opts, mode, enum_dev, cap, roots_dev, n_roots_list, root_counts_dev, out);
}

tm_status check_graph_args(const uint32_t *src, const uint32_t *dst, const int64_t *t, uint64_t m, uint32_t n,
                           tm_graph **out) {
    if (!out) return fail(TM_EINVAL, "out is null");
    *out = nullptr;
    if (m > TM_MAX_M) return fail(TM_EINVAL, "m exceeds TM_MAX_M (2^31-1)");
    if (m + (uint64_t)n > (1ull << 31) - 4) return fail(TM_EINVAL, "m + n_vertices must stay below 2^31 - 4");
    if (m && (!src || !dst || !t)) return fail(TM_EINVAL, "null edge array");
    if (m && n == 0) return fail(TM_EINVAL, "n_vertices is 0 but m > 0");
    return TM_OK;
}

}  // namespace
}  // namespace tmg

using namespace tmg;

extern "C" {

const char *tm_last_error(void) { return g_err.c_str(); }
const char *tm_version(void) { return "tmotif 0.1 (sm_100a)"; }

void tm_run_opts_default(tm_run_opts *o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->root_lo = 0;
    o->root_hi = UINT64_MAX;
}

tm_status tm_graph_create(const uint32_t *src, const uint32_t *dst, const int64_t *t, uint64_t m,
                          uint32_t n_vertices, const tm_graph_opts *o, tm_graph **out) {
    g_err.clear();
    tm_status st = check_graph_args(src, dst, t, m, n_vertices, out);
    if (st) return st;
    if (!(o && o->input_on_device) && m <= (1u << 20)) {  // small host input: exact messages here; the device check covers the rest
        for (uint64_t i = 0; i < m; i++) {
            if (src[i] >= n_vertices || dst[i] >= n_vertices)
                return fail(TM_EINVAL, "edge " + std::to_string(i) + ": endpoint >= n_vertices");
            if (t[i] < 0) return fail(TM_EINVAL, "edge " + std::to_string(i) + ": negative timestamp");
        }
    }
    DeviceGuard guard(o ? o->device : -1);
    return graph_create(src, dst, t, m, n_vertices, o, out);
}

tm_status tm_graph_destroy(tm_graph *g) {
    graph_destroy(g);
    return TM_OK;
}

tm_status tm_graph_info(const tm_graph *g, uint64_t *m, uint32_t *n, int *device) {
    if (!g) return fail(TM_EINVAL, "null graph");
    if (m) *m = g->d.m;
    if (n) *n = g->d.n;
    if (device) *device = g->device;
    return TM_OK;
}

tm_status tm_graph_sorted_to_input(const tm_graph *g, uint64_t *perm) {
    if (!g || (!perm && g->d.m)) return fail(TM_EINVAL, "null argument");
    DeviceGuard guard(g->device);
    std::vector<uint32_t> tmp(g->d.m);
    if (g->d.m) TM_CUDA_TRY(cudaMemcpy(tmp.data(), g->d.perm, g->d.m * 4, cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < g->d.m; i++) perm[i] = tmp[i];
    return TM_OK;
}

tm_status tm_graph_sorted_edges(const tm_graph *g, uint32_t *src, uint32_t *dst, int64_t *t) {
    if (!g) return fail(TM_EINVAL, "null graph");
    DeviceGuard guard(g->device);
    const uint64_t m = g->d.m;
    if (!m) return TM_OK;
    if (src) TM_CUDA_TRY(cudaMemcpy(src, g->d.src, m * 4, cudaMemcpyDeviceToHost));
    if (dst) TM_CUDA_TRY(cudaMemcpy(dst, g->d.dst, m * 4, cudaMemcpyDeviceToHost));
    if (t) TM_CUDA_TRY(cudaMemcpy(t, g->d.t, m * 8, cudaMemcpyDeviceToHost));
    return TM_OK;
}

tm_status tm_motif_create(uint32_t L, const uint32_t *mu, const uint32_t *mv, int64_t delta, const int64_t *fine,
                          tm_motif **out) {
    g_err.clear();
    if (!out) return fail(TM_EINVAL, "out is null");
    *out = nullptr;
    if (L < 1 || L > TM_MAX_EDGES) return fail(TM_EINVAL, "L must be in 1..TM_MAX_EDGES");
    if (!mu || !mv) return fail(TM_EINVAL, "null motif edge array");
    if (delta < 0) return fail(TM_EINVAL, "delta < 0");
    int label[64];
    for (int &x : label) x = -1;
    int nv = 0;
    tm_motif mo;
    mo.L = L;
    mo.delta = delta;
    for (uint32_t i = 0; i < L; i++) {
        if (mu[i] >= 64 || mv[i] >= 64) return fail(TM_EINVAL, "motif vertex label >= 64");
        if (mu[i] == mv[i]) return fail(TM_EINVAL, "motif self-loop");
        const bool seen_u = label[mu[i]] >= 0, seen_v = label[mv[i]] >= 0;
        if (i > 0 && !seen_u && !seen_v) mo.disconnected = true;   // AllEdges candidates (Q9)
        // relabel by first appearance (u before v)
        if (!seen_u) label[mu[i]] = nv++;
        if (!seen_v) label[mv[i]] = nv++;
        if (nv > TM_MAX_VERTICES) return fail(TM_EINVAL, "more than TM_MAX_VERTICES motif vertices");
        mo.u[i] = (uint8_t)label[mu[i]];
        mo.v[i] = (uint8_t)label[mv[i]];
    }
    mo.nv = nv;
    for (int i = 0; i < 64; i++) mo.internal[i] = (int8_t)label[i];
    for (int i = 0; i < kMaxV; i++) mo.vreq[i] = TM_ANY_LABEL;
    for (int i = 0; i < kMaxL; i++) mo.ereq[i] = TM_ANY_LABEL;
    for (int i = 0; i < kMaxL; i++) mo.fine[i] = TM_DELTA_INF;
    if (fine)
        for (uint32_t i = 0; i + 1 < L; i++) {
            if (fine[i] < 0) return fail(TM_EINVAL, "fine delta < 0");
            mo.fine[i] = fine[i];
        }
    mo.code = motif_code((int)L, mo.u, mo.v);
    tm_motif *p = new (std::nothrow) tm_motif(mo);
    if (!p) return fail(TM_ENOMEM, "host allocation failed");
    *out = p;
    return TM_OK;
}

tm_status tm_motif_destroy(tm_motif *mo) {
    delete mo;
    return TM_OK;
}

tm_status tm_motif_set_vertex_label(tm_motif *mo, uint32_t vertex, int32_t label) {
    g_err.clear();
    if (!mo || vertex >= 64 || mo->internal[vertex] < 0) return fail(TM_EINVAL, "vertex is not in the motif");
    if (label < TM_ANY_LABEL) return fail(TM_EINVAL, "label < -1");
    mo->vreq[mo->internal[vertex]] = label;
    mo->rtc_fn[0] = mo->rtc_fn[1] = nullptr;   // a specialisation no longer fits: re-run tm_motif_specialise
    return TM_OK;
}

tm_status tm_motif_set_edge_label(tm_motif *mo, uint32_t edge, int32_t label) {
    g_err.clear();
    if (!mo || edge >= mo->L) return fail(TM_EINVAL, "edge >= L");
    if (label < TM_ANY_LABEL) return fail(TM_EINVAL, "label < -1");
    mo->ereq[edge] = label;
    mo->rtc_fn[0] = mo->rtc_fn[1] = nullptr;
    return TM_OK;
}

tm_status tm_motif_add_anti_edge(tm_motif *mo, uint32_t u, uint32_t v, uint32_t attach, int64_t window) {
    g_err.clear();
    if (!mo) return fail(TM_EINVAL, "null motif");
    if (mo->n_anti >= TM_MAX_ANTI) return fail(TM_EINVAL, "more than TM_MAX_ANTI anti-edges");
    if (u >= 64 || v >= 64 || mo->internal[u] < 0 || mo->internal[v] < 0 || u == v)
        return fail(TM_EINVAL, "anti-edge endpoints must be distinct motif vertices");
    if (attach >= mo->L) return fail(TM_EINVAL, "attach >= L");
    if (window < 0 || window == TM_DELTA_INF) return fail(TM_EINVAL, "anti-edge window must be finite and >= 0");
    const uint32_t j = mo->n_anti++;
    mo->anti_u[j] = (uint8_t)mo->internal[u];
    mo->anti_v[j] = (uint8_t)mo->internal[v];
    mo->anti_attach[j] = (uint8_t)attach;
    mo->anti_window[j] = window;
    mo->rtc_fn[0] = mo->rtc_fn[1] = nullptr;
    return TM_OK;
}

tm_status tm_graph_set_labels(tm_graph *g, const int32_t *vlabels, const int32_t *elabels, int on_device) {
    g_err.clear();
    if (!g) return fail(TM_EINVAL, "null graph");
    DeviceGuard guard(g->device);
    return set_labels(g->d, vlabels, elabels, on_device != 0);
}

tm_status tm_motif_specialised(const tm_motif *mo, int *sp) {
    if (!mo || !sp) return fail(TM_EINVAL, "null argument");
    *sp = !mo->disconnected && (mo->rtc_fn[kCount] || (is_specialised(mo->code) && !mo->constrained())) ? 1 : 0;
    return TM_OK;
}

tm_status tm_motif_specialise(tm_motif *mo) {
    g_err.clear();
    if (!mo) return fail(TM_EINVAL, "null motif");
    if (mo->disconnected) return fail(TM_EUNSUPPORTED, "a prefix-disconnected motif (Q9) runs the dfs kernel");
    if (is_specialised(mo->code) && !mo->constrained()) return TM_OK;   // in the build-time catalog
    for (int mode : {(int)kCount, (int)kEnum}) {
        RtcKernel k;
        const tm_status st = rtc_kernel(mo->code, mo->constrained(), mode, &k);
        if (st) return st;
        mo->rtc_fn[mode] = k.fn;
        mo->rtc_smem[mode] = k.smem_per_warp;
    }
    return TM_OK;
}

tm_status tm_count(const tm_graph *g, const tm_motif *mo, const tm_run_opts *o, uint64_t *count) {
    g_err.clear();
    if (!count) return fail(TM_EINVAL, "count is null");
    RunOut r;
    tm_status st = run(g, mo, o, kCount, nullptr, 0, nullptr, 0, nullptr, &r);
    if (st) return st;
    *count = r.count;
    return TM_OK;
}

tm_status tm_search_stats_run(const tm_graph *g, const tm_motif *mo, const tm_run_opts *o, tm_search_stats *out) {
    g_err.clear();
    if (!out) return fail(TM_EINVAL, "out is null");
    RunOut r;
    tm_status st = run(g, mo, o, kStats, nullptr, 0, nullptr, 0, nullptr, &r);
    if (st) return st;
    std::memset(out, 0, sizeof *out);
    for (int l = 0; l < kMaxL && l < 8; l++) out->nodes[l] = r.stats[kStatsBase + l];
    // roots that bind motif edge 1 are the level-1 nodes when L >= 2
    out->window_sum = r.stats[16];
    out->list_sum = r.stats[17];
    out->probe_sum = r.stats[18];
    out->fast_window_sum = r.stats[19];
    out->matches = r.count;
    return TM_OK;
}

tm_status tm_enumerate(const tm_graph *g, const tm_motif *mo, const tm_run_opts *o, uint32_t *buf, uint64_t cap,
                       uint64_t *n_total, uint64_t *n_written) {
    g_err.clear();
    if (!g || !mo || !n_total) return fail(TM_EINVAL, "null argument");
    if (cap && !buf) return fail(TM_EINVAL, "buf is null with cap > 0");
    tm_run_opts opt;
    tm_run_opts_default(&opt);
    if (o) opt = *o;
    DeviceGuard guard(g->device);
    cudaStream_t s = (cudaStream_t)opt.stream;
    const uint32_t L = mo->L;
    uint32_t *dbuf = buf;
    if (!opt.buffers_on_device && cap) TM_CUDA_TRY(dev_alloc((void **)&dbuf, cap * L * sizeof(uint32_t), s));
    RunOut r;
    tm_status st = run(g, mo, &opt, kEnum, dbuf, cap, nullptr, 0, nullptr, &r);
    const uint64_t written = std::min(r.count, cap);
    if (st == TM_OK && written && (opt.canonical || !opt.buffers_on_device)) {
        std::vector<uint32_t> rows(written * L);
        cudaError_t e = cudaMemcpyAsync(rows.data(), dbuf, written * L * 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = fail(TM_ECUDA, std::string("enumeration copy: ") + cudaGetErrorString(e));
        if (st == TM_OK && opt.canonical) {
            std::vector<uint64_t> idx(written);
            for (uint64_t i = 0; i < written; i++) idx[i] = i;
            std::sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
                return std::lexicographical_compare(&rows[a * L], &rows[a * L + L], &rows[b * L], &rows[b * L + L]);
            });
            std::vector<uint32_t> sorted(written * L);
            for (uint64_t i = 0; i < written; i++) std::memcpy(&sorted[i * L], &rows[idx[i] * L], L * 4);
            rows.swap(sorted);
        }
        if (st == TM_OK) {
            if (opt.buffers_on_device) {
                e = cudaMemcpyAsync(dbuf, rows.data(), written * L * 4, cudaMemcpyHostToDevice, s);
                if (e == cudaSuccess) e = cudaStreamSynchronize(s);
                if (e != cudaSuccess) st = fail(TM_ECUDA, std::string("enumeration copy: ") + cudaGetErrorString(e));
            } else {
                std::memcpy(buf, rows.data(), written * L * 4);
            }
        }
    }
    if (!opt.buffers_on_device && cap) { dev_free(dbuf, s); cudaStreamSynchronize(s); }
    if (st) return st;
    *n_total = r.count;
    if (n_written) *n_written = written;
    if (r.count > cap) return fail(TM_TRUNCATED, "more matches than buffer rows");
    return TM_OK;
}

tm_status tm_count_roots(const tm_graph *g, const tm_motif *mo, const tm_run_opts *o, const uint64_t *roots,
                         uint64_t n, uint64_t *counts) {
    g_err.clear();
    if (!g || !mo || (n && (!roots || !counts))) return fail(TM_EINVAL, "null argument");
    tm_run_opts opt;
    tm_run_opts_default(&opt);
    if (o) opt = *o;
    if (n == 0) return TM_OK;
    if (n >= (1ull << 32)) return fail(TM_EINVAL, "more than 2^32 - 1 roots in one call");
    DeviceGuard guard(g->device);
    cudaStream_t s = (cudaStream_t)opt.stream;
    const uint64_t *droots = roots;
    unsigned long long *dcounts = reinterpret_cast<unsigned long long *>(counts);
    uint64_t *own_r = nullptr;
    unsigned long long *own_c = nullptr;
    if (!opt.buffers_on_device) {
        for (uint64_t i = 0; i < n; i++)
            if (roots[i] >= g->d.m) return fail(TM_EINVAL, "root id >= m");
        TM_CUDA_TRY(dev_alloc((void **)&own_r, n * 8, s));
        TM_CUDA_TRY(dev_alloc((void **)&own_c, n * 8, s));
        TM_CUDA_TRY(cudaMemcpyAsync(own_r, roots, n * 8, cudaMemcpyHostToDevice, s));
        droots = own_r;
        dcounts = own_c;
    }
    TM_CUDA_TRY(cudaMemsetAsync(dcounts, 0, n * 8, s));
    RunOut r;
    tm_status st = run(g, mo, &opt, kRoots, nullptr, 0, droots, n, dcounts, &r);
    if (st == TM_OK && !opt.buffers_on_device) {
        cudaError_t e = cudaMemcpyAsync(counts, own_c, n * 8, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = fail(TM_ECUDA, std::string("counts copy: ") + cudaGetErrorString(e));
    }
    dev_free(own_r, s);
    dev_free(own_c, s);
    cudaStreamSynchronize(s);
    return st;
}

tm_status tm_census36(const tm_graph *g, int64_t delta, const int64_t *fine, const tm_run_opts *o,
                      uint64_t *counts) {
    g_err.clear();
    if (!g || !counts) return fail(TM_EINVAL, "null argument");
    if (delta < 0) return fail(TM_EINVAL, "delta < 0");
    if (fine && (fine[0] < 0 || fine[1] < 0)) return fail(TM_EINVAL, "fine delta < 0");
    tm_run_opts opt;
    tm_run_opts_default(&opt);
    if (o) opt = *o;
    DeviceGuard guard(g->device);
    cudaStream_t s = (cudaStream_t)opt.stream;
    const DeviceGraph &d = g->d;
    const uint64_t m = d.m;
    g_info = tm_run_info{};
    CensusParams p;
    std::memset(&p, 0, sizeof p);
    p.src = d.src; p.dst = d.dst; p.rec = d.rec; p.rank = d.rank; p.m = (uint32_t)m;
    const uint64_t hi = std::min<uint64_t>(opt.root_hi, m), lo = std::min<uint64_t>(opt.root_lo, hi);
    p.root_lo = lo;
    p.n_roots = hi - lo;
    // distinct horizons: δ, then δ_1, δ_2 when finite and < δ (a larger gap bound never binds)
    std::vector<int64_t> hv{delta};
    int gi[2] = {-1, -1};
    for (int i = 0; i < 2 && fine; i++) {
        if (fine[i] == TM_DELTA_INF || fine[i] >= delta) continue;
        auto it = std::find(hv.begin(), hv.end(), fine[i]);
        gi[i] = (int)(it - hv.begin());
        if (it == hv.end()) hv.push_back(fine[i]);
    }
    unsigned long long *dcounts = nullptr;
    uint32_t *hbuf = nullptr;
    const uint64_t mh = (m + 3) & ~3ull;   // horizon stride: 16-byte aligned arrays (vector stores)
    TM_CUDA_TRY(dev_alloc((void **)&dcounts, 36 * sizeof(unsigned long long), s));
    struct Free {
        void *a, *b, *c;
        cudaStream_t s;
        ~Free() { dev_free(a, s); dev_free(b, s); dev_free(c, s); }
    } fr{dcounts, nullptr, nullptr, s};
    TM_CUDA_TRY(cudaMemsetAsync(dcounts, 0, 36 * sizeof(unsigned long long), s));
    p.counts = dcounts;
    cudaEvent_t ev[4] = {};
    for (auto &e : ev) TM_CUDA_TRY(cudaEventCreate(&e));
    struct EvFree { cudaEvent_t *e; ~EvFree() { for (int i = 0; i < 4; i++) if (e[i]) cudaEventDestroy(e[i]); } } evf{ev};
    TM_CUDA_TRY(cudaEventRecord(ev[0], s));
    if (p.n_roots > 0) {
        TM_CUDA_TRY(dev_alloc((void **)&hbuf, hv.size() * mh * sizeof(uint32_t), s));
        fr.b = hbuf;
        for (size_t i = 0; i < hv.size(); i += 2) {
            const bool two = i + 1 < hv.size();
            TM_CUDA_TRY(build_horizons(d, hv[i], two ? hv[i + 1] : hv[i], hbuf + i * mh,
                                       two ? hbuf + (i + 1) * mh : nullptr, s));
            g_info.launches += 2;
        }
        p.H = hbuf;
        p.Hf0 = gi[0] >= 0 ? hbuf + (size_t)gi[0] * mh : nullptr;
        p.Hf1 = gi[1] >= 0 ? hbuf + (size_t)gi[1] * mh : nullptr;
    }
    TM_CUDA_TRY(cudaEventRecord(ev[1], s));
    if (p.n_roots > 0) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        TM_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const uint64_t want = (p.n_roots + 255) / 256;
        const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)sms * 8));
        TM_CUDA_TRY(launch_census36(p, grid, s));
        g_info.launches++;
        g_info.grid_ctas = (uint32_t)grid;
        g_info.block_threads = 256;
    }
    TM_CUDA_TRY(cudaEventRecord(ev[2], s));
    unsigned long long host[36];
    TM_CUDA_TRY(cudaMemcpyAsync(host, dcounts, sizeof host, cudaMemcpyDeviceToHost, s));
    TM_CUDA_TRY(cudaEventRecord(ev[3], s));
    TM_CUDA_TRY(cudaStreamSynchronize(s));
    cudaEventElapsedTime(&g_info.horizon_ms, ev[0], ev[1]);
    cudaEventElapsedTime(&g_info.mine_ms, ev[1], ev[2]);
    cudaEventElapsedTime(&g_info.total_ms, ev[0], ev[3]);
    for (int i = 0; i < 36; i++) counts[i] = host[i];
    return TM_OK;
}

tm_status tm_count_multi(const tm_graph *g, const tm_motif *const *mos, uint32_t k, const tm_run_opts *o,
                         uint64_t *counts) {
    g_err.clear();
    if (!counts || !mos || k == 0) return fail(TM_EINVAL, "null argument or k == 0");
    std::vector<RunOut> r(k);
    tm_status st = run_multi(g, mos, k, o, kCount, nullptr, 0, nullptr, 0, nullptr, r.data());
    if (st) return st;
    for (uint32_t i = 0; i < k; i++) counts[i] = r[i].count;
    return TM_OK;
}

tm_status tm_last_kernel_info(tm_kernel_info *out, uint32_t cap, uint32_t *n) {
    if (!n || (cap && !out)) return fail(TM_EINVAL, "null argument");
    *n = (uint32_t)g_kinfo.size();
    for (uint32_t i = 0; i < cap && i < g_kinfo.size(); i++) out[i] = g_kinfo[i];
    return TM_OK;
}

tm_status tm_last_run_info(tm_run_info *out) {
    if (!out) return fail(TM_EINVAL, "out is null");
    *out = g_info;
    return TM_OK;
}

tm_status tm_partition_plan(const int64_t *t, uint64_t m, int64_t delta, uint32_t P, const uint64_t *weights,
                            uint64_t *root_lo, uint64_t *edge_hi) {
    g_err.clear();
    if (P == 0 || !root_lo || !edge_hi || (m && !t)) return fail(TM_EINVAL, "bad argument");
    if (delta < 0) return fail(TM_EINVAL, "delta < 0");
    for (uint64_t i = 0; i + 1 < m; i++)
        if (t[i] > t[i + 1]) return fail(TM_EINVAL, "t_sorted is not sorted");
    auto horizon = [&](uint64_t r) -> uint64_t {  // max{j : t[j] <= t[r] + δ}
        if (delta == TM_DELTA_INF || t[r] > INT64_MAX - delta) return m - 1;
        return (uint64_t)(std::upper_bound(t + r, t + m, t[r] + delta) - t) - 1;
    };
    std::vector<long double> pre(m + 1, 0.0L);
    for (uint64_t r = 0; r < m; r++)
        pre[r + 1] = pre[r] + (long double)(weights ? weights[r] : (horizon(r) - r + 1));
    root_lo[0] = 0;
    for (uint32_t q = 1; q < P; q++) {
        long double target = pre[m] * q / P;
        uint64_t r = (uint64_t)(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
        r = std::min<uint64_t>(r, m);
        // cut only where the timestamp changes: a rank's slice then starts at
        // the first edge of its timestamp, so every edge with t >= t(root_lo)
        // is in it — an anti-edge witness tied with the slice's first root
        // (window [t(e_a), ...]) is never cut off
        if (r < m) r = (uint64_t)(std::lower_bound(t, t + m, t[r]) - t);
        r = std::max<uint64_t>(r, root_lo[q - 1]);
        root_lo[q] = r;
    }
    root_lo[P] = m;
    for (uint32_t q = 0; q < P; q++)
        edge_hi[q] = root_lo[q + 1] > root_lo[q] ? horizon(root_lo[q + 1] - 1) + 1 : root_lo[q];
    return TM_OK;
}

}  // extern "C"
