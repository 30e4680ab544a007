// nnc/geometry.hpp -- spatial geometry, integer-exact with the reference
// (kernels.cpp:12-53): TF-SAME out = ceil(in/s), pad_top = max((o-1)s+k-in,0)/2
// (extra pad on the bottom/right); VALID out = (in-k)/s+1; MaxPool is VALID only.
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

#include "nncb.h"
#include "nnc/error.hpp"
#include "nnc/hlir.hpp"

namespace nnc::geom {

inline int64_t window_out_extent(int64_t in, int64_t k, int64_t s, hlir::Padding p) {
    if (p == hlir::Padding::Same) return (in + s - 1) / s;
    if (in < k) throw Error(Error::Code::ExtentMismatch, "window larger than input extent");
    return (in - k) / s + 1;
}

/// Fills the conv fields of a GEMM descriptor from an NHWC input shape.
inline void conv_geometry(nncb_gemm_desc& d, const std::vector<int64_t>& x, const hlir::Attrs& a) {
    if (x.size() != 4) throw Error(Error::Code::RankError, "conv: rank-4 NHWC input required");
    d.n = x[0]; d.ih = x[1]; d.iw = x[2]; d.ci = x[3];
    d.co = a.out_channels; d.kh = a.kernel[0]; d.kw = a.kernel[1];
    d.sh = a.stride[0]; d.sw = a.stride[1];
    d.oh = window_out_extent(d.ih, d.kh, d.sh, a.padding);
    d.ow = window_out_extent(d.iw, d.kw, d.sw, a.padding);
    d.pad_top = d.pad_left = 0;
    if (a.padding == hlir::Padding::Same) {
        d.pad_top = std::max<int64_t>((d.oh - 1) * d.sh + d.kh - d.ih, 0) / 2;
        d.pad_left = std::max<int64_t>((d.ow - 1) * d.sw + d.kw - d.iw, 0) / 2;
    }
}

inline nncb_pool_geom pool_geometry(const std::vector<int64_t>& x, const hlir::Attrs& a) {
    if (x.size() != 4) throw Error(Error::Code::RankError, "pool: rank-4 NHWC input required");
    nncb_pool_geom g{};
    g.n = x[0]; g.ih = x[1]; g.iw = x[2]; g.c = x[3];
    g.kh = a.kernel[0]; g.kw = a.kernel[1]; g.sh = a.stride[0]; g.sw = a.stride[1];
    g.oh = window_out_extent(g.ih, g.kh, g.sh, hlir::Padding::Valid);
    g.ow = window_out_extent(g.iw, g.kw, g.sw, hlir::Padding::Valid);
    return g;
}

}  // namespace nnc::geom
