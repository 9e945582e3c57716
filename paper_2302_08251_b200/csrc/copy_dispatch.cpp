// copyView dispatch (view.cpp:168-189) and the host-buffer entry point.
#include "capi_internal.hpp"

#include <cstdlib>
#include <cstring>

using namespace lamb;

namespace lamhost
{
    static uint64_t gcd64(uint64_t a, uint64_t b)
    {
        while(b)
        {
            const uint64_t t = a % b;
            a = b;
            b = t;
        }
        return a;
    }

    static bool sameLayout(const Map& a, const Map& b)
    {
        // view.cpp:175-176
        return a.name() == b.name() && !a.hasMutableState() && !b.hasMutableState() && a.isFullyPhysical()
            && b.isFullyPhysical();
    }

    void copyViews(const lam_view& src, lam_view& dst, uint64_t begin, uint64_t end, cudaStream_t s)
    {
        const Map& a = *src.L->map;
        const Map& b = *dst.L->map;
        if(!(a.schema() == b.schema()) || !(a.extents() == b.extents()))
            throw std::invalid_argument("incompatible views");
        if(src.device != dst.device)
            throw std::invalid_argument("views live on different devices");
        const uint64_t n = a.elementCount();
        if(begin > end || end > n)
            throw std::out_of_range("index out of range: elements [" + std::to_string(begin) + ", " + std::to_string(end) + ")");
        const bool full = begin == 0 && end == n;
        if(!full)
        {
            const uint64_t u1 = src.L->shardUnit, u2 = dst.L->shardUnit;
            const uint64_t unit = u1 / gcd64(u1, u2) * u2;
            if(begin % unit != 0 || (end != n && end % unit != 0))
                throw std::invalid_argument("copy range must start (and end, unless at the element count) on a "
                                            "multiple of the shard unit " + std::to_string(unit));
        }
        if(begin == end || a.schema().leafCount() == 0)
            return;
        DeviceGuard g(src.device);
        // LAMB_FORCE_TILE=1 (profiling only) routes equal layouts through the tile engine
        static const bool forceTile = std::getenv("LAMB_FORCE_TILE") && std::getenv("LAMB_FORCE_TILE")[0] == '1';
        if(full && sameLayout(a, b) && !forceTile)
        {
            for(size_t nr = 0; nr < a.blobCount(); ++nr)
                lam_cuda_check(lamk::blob_copy(dst.blobs[nr], src.blobs[nr], a.blobSize(nr), s), "blob_copy");
            return;
        }
        // LAMB_FORCE_GENERIC=1 (tests only): cross-check the specialised kernels against the
        // plan interpreter on identical inputs
        const char* fg = std::getenv("LAMB_FORCE_GENERIC");
        if(!(fg && fg[0] == '1') && tileCopy(src, dst, begin, end, s))
            return;
        lam_cuda_check(lamk::generic_copy(src.img.hdr, dst.img.hdr, begin, end,
                                          static_cast<uint32_t>(a.schema().leafCount()), src.L->fac, dst.L->fac, s),
                       "generic_copy");
    }

    void copyHost(const lam_layout& sl, const void* const* sb, const lam_layout& dl, void* const* db, int device,
                  uint64_t* srcCounters, uint64_t* dstCounters)
    {
        const Map& a = *sl.L->map;
        const Map& b = *dl.L->map;
        if(!(a.schema() == b.schema()) || !(a.extents() == b.extents()))
            throw std::invalid_argument("incompatible views");
        DeviceGuard g(device);
        HostPipeline& hp = HostPipeline::get(device);
        hp.run(sl, sb, dl, db, srcCounters, dstCounters);
    }
} // namespace lamhost
