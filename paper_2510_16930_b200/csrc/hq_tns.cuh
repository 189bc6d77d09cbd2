// hq_tns.cuh — parsed `.tns` contents behind the C-ABI handle (hq_tns.cu)
#pragma once

#include <cstdint>
#include <vector>

struct hq_tns {
    int order = 0;
    std::vector<uint64_t> dims;
    std::vector<uint32_t> coords;  // nnz x order, file order
    std::vector<double> values;
};
