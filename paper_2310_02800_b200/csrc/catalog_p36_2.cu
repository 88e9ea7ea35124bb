#include "catalog.cuh"

namespace tmg {

namespace {
template <int... I>
void add(std::vector<CatalogEntry> &v, std::integer_sequence<int, I...>) {
    (v.push_back(entry<p36_code<I + 2 * 9>()>()), ...);
}
}  // namespace

template <>
void register_p36_part<2>(std::vector<CatalogEntry> &v) { add(v, std::make_integer_sequence<int, 9>{}); }

}  // namespace tmg
