#include "catalog.cuh"

namespace tmg {

void register_named(std::vector<CatalogEntry> &v) {
    v.push_back(entry<mcode(1, 0, 1)>());                               // single edge
    v.push_back(entry<mcode(2, 0, 1, 1, 2)>());                         // 2-path
    // motifs of >= 3 edges also carry a prefix-fusion counting kernel
    // (tm_count_multi counts their prefixes, e.g. P3 inside C4, TRI inside DIA)
    v.push_back(entry<mcode(3, 0, 1, 1, 2, 2, 3), true>());             // P3   3-path
    v.push_back(entry<mcode(3, 0, 1, 0, 2, 0, 3), true>());             // STAR3 out-star
    v.push_back(entry<mcode(4, 0, 1, 1, 2, 2, 3, 3, 0), true>());       // C4   4-cycle
    v.push_back(entry<mcode(4, 0, 1, 1, 2, 2, 0, 0, 3), true>());       // TT   tailed triangle
    v.push_back(entry<mcode(4, 0, 1, 1, 2, 2, 3, 3, 1), true>());       // TT2  tailed triangle, tail first
    v.push_back(entry<mcode(5, 0, 1, 1, 2, 2, 0, 1, 3, 3, 2), true>()); // DIA  diamond
}

}  // namespace tmg
