// Greedy graph colouring shared by the factorization's level colouring and
// the h2f_greedy_coloring entry point (structure.py:137-167): vertices in the
// given order, each takes the smallest colour none of its already-coloured
// neighbours has.  `for_each_nbr(i, visit)` calls visit(j) for every
// neighbour position j of vertex i.
#pragma once
#include <algorithm>
#include <vector>

namespace h2f {

template <class NbrFn>
int greedy_coloring(const std::vector<size_t>& order, size_t nv, NbrFn for_each_nbr, std::vector<int>& color) {
    color.assign(nv, -1);
    int ncolors = 0;
    std::vector<char> used;
    for (size_t i : order) {
        used.clear();
        for_each_nbr(i, [&](size_t j) {
            const int cj = color[j];
            if (cj >= 0) {
                if (size_t(cj) >= used.size()) used.resize(cj + 1, 0);
                used[cj] = 1;
            }
        });
        int c = 0;
        while (size_t(c) < used.size() && used[c]) ++c;
        color[i] = c;
        ncolors = std::max(ncolors, c + 1);
    }
    return ncolors;
}

}  // namespace h2f
