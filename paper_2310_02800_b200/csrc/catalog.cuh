// Kernel catalog: compile-time specialised instantiations of mine_kernel for
// the named motifs (the B200 counterpart of the paper's motif-specific code
// generation), plus the generic runtime-plan kernel.
#pragma once

#include <vector>

#include "mine.cuh"

namespace tmg {

constexpr uint64_t mcode(int L, int a0, int b0, int a1 = 0, int b1 = 0, int a2 = 0, int b2 = 0, int a3 = 0,
                         int b3 = 0, int a4 = 0, int b4 = 0, int a5 = 0, int b5 = 0) {
    const int a[6] = {a0, a1, a2, a3, a4, a5}, b[6] = {b0, b1, b2, b3, b4, b5};
    uint64_t c = (uint64_t)L;
    for (int i = 0; i < L; i++) c |= ((uint64_t)a[i] << (3 + 6 * i)) | ((uint64_t)b[i] << (6 + 6 * i));
    return c;
}

struct CatalogEntry {
    uint64_t code;
    KernelInfo count, enumerate;
    KernelInfo count_pfx;   // counting + prefix fusion / sibling emission (named motifs); fn == nullptr: none
    KernelInfo resume;      // counting resumed from rows of partial matches (named motifs)
    KernelInfo count_sib;   // kCountPfx + sibling rows at level 2 (named motifs of >= 4 edges)
};

template <uint64_t CODE, bool PFX = false>
CatalogEntry entry() {
    KernelInfo pfx{nullptr, 0}, res{nullptr, 0}, sib{nullptr, 0};
    if constexpr (PFX) {
        pfx = kernel_info<PlanC<CODE>, kCountPfx>();
        res = kernel_info<PlanC<CODE>, kResume>();
        if constexpr (PlanC<CODE>::kL >= 4) sib = kernel_info<PlanC<CODE>, kCountSib>();
    }
    return CatalogEntry{CODE, kernel_info<PlanC<CODE>, kCount>(), kernel_info<PlanC<CODE>, kEnum>(), pfx, res, sib};
}

void register_named(std::vector<CatalogEntry> &v);
template <int P>
void register_p36_part(std::vector<CatalogEntry> &v);
constexpr int kP36Parts = 4;

// Paranjape's 36 motifs (0->1, E[a], E[b]), E = [01, 10, 02, 20, 12, 21]
constexpr int kE6[6][2] = {{0, 1}, {1, 0}, {0, 2}, {2, 0}, {1, 2}, {2, 1}};
template <int I>
constexpr uint64_t p36_code() {
    return mcode(3, 0, 1, kE6[I / 6][0], kE6[I / 6][1], kE6[I % 6][0], kE6[I % 6][1]);
}

}  // namespace tmg
