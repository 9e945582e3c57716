// Tile-engine eligibility and launch (filled in by copy_tile.cu's host side).
#include "capi_internal.hpp"

namespace lamhost
{
    bool tileCopyImages(const lamb::Lowered&, const DeviceImage&, const lamb::Lowered&, DeviceImage&, uint64_t,
                        uint64_t, cudaStream_t)
    {
        return false;
    }

    bool tileCopy(const lam_view& src, lam_view& dst, uint64_t begin, uint64_t end, cudaStream_t s)
    {
        return tileCopyImages(*src.L, src.img, *dst.L, dst.img, begin, end, s);
    }
} // namespace lamhost
