// ConvGeometry — same fields, floor rule and validation as the reference
// (proj/include/portten/conv_geometry.hpp:28-75); convertible to the C-ABI descriptor.
#pragma once

#include <cstdint>
#include <string>

#include "../pt_b200.h"
#include "portten/errors.hpp"

namespace portten::conv {

struct ConvGeometry {
    std::int64_t batch = 1;
    std::int64_t inChannels = 1;
    std::int64_t inHeight = 1;
    std::int64_t inWidth = 1;
    std::int64_t outChannels = 1;
    std::int64_t kernelH = 1;
    std::int64_t kernelW = 1;
    std::int64_t padH = 0;
    std::int64_t padW = 0;
    std::int64_t strideH = 1;
    std::int64_t strideW = 1;

    std::int64_t outHeight() const { return (inHeight + 2 * padH - kernelH) / strideH + 1; }
    std::int64_t outWidth() const { return (inWidth + 2 * padW - kernelW) / strideW + 1; }
    std::int64_t patchSize() const { return inChannels * kernelH * kernelW; }
    std::int64_t outSpatial() const { return outHeight() * outWidth(); }

    void validate() const;
    std::string toString() const;
    pt_conv_geom abi() const {
        return pt_conv_geom{batch, inChannels, inHeight, inWidth, outChannels, kernelH, kernelW,
                            padH, padW, strideH, strideW};
    }
    bool operator==(const ConvGeometry&) const = default;
};

}  // namespace portten::conv
