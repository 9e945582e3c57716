// Maintainer-side binding: lamina::copyViewB200 for the reference's own host views.
//
// This header is what a lamina maintainer adds to the reference.  It
// includes the reference's headers (<lamina/lamina.hpp>, /root/reference/proj/core/include)
// and the C ABI of this repo (lamina_b200.h); nothing else.  It is compiled and exercised by
// oracle/Makefile (target binding_check) against the reference, and run as a GPU test
// (tests/test_gpu_binding.py) next to lamina::copyView on the same lamina::View objects.
//
// Lowering: every mapping the reference's layout grammar can build prints itself through
// Mapping::name() (wrappers included: "field-access-count(...)", "heatmap:g(...)"), and the
// schema / extents through RecordSchema::toString / ArrayExtents::toString, so the binding
// needs no access to lamina internals.  A user-defined Mapping subclass (mapping.hpp:44-155)
// has a name the grammar does not know: lowering fails with std::invalid_argument
// ("copyViewB200: mapping '<name>' cannot be lowered ...") and the caller keeps using
// lamina::copyView for it.
#pragma once

#include <lamina/lamina.hpp>

#include "lamina_b200.h"

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace lamina
{
    /// Counter deltas of one copyViewB200 call, per side: FieldAccessCount reads/writes per
    /// flat leaf (instrument.hpp:11-21), then Heatmap block counters per blob in blob order.
    /// The reference keeps its counters private (instrument.hpp:54-65: counters(), reset(),
    /// no add), so they are handed back here instead of being added into the mapping.
    struct B200CopyCounters
    {
        std::vector<std::uint64_t> srcReads, srcWrites, dstReads, dstWrites;
        std::vector<std::vector<std::uint64_t>> srcHeat, dstHeat;
    };

    namespace b200_detail
    {
        [[noreturn]] inline void rethrow(int rc)
        {
            const std::string msg = lam_last_error();
            switch(rc)
            {
            case LAM_EINVAL:
                throw std::invalid_argument(msg);
            case LAM_ERANGE:
                throw std::out_of_range(msg);
            case LAM_EOVERFLOW:
                throw std::overflow_error(msg);
            case LAM_ELOGIC:
                throw std::logic_error(msg);
            default:
                throw std::runtime_error(msg);
            }
        }

        struct Lowered
        {
            lam_layout* h = nullptr;
            ~Lowered()
            {
                if(h)
                    lam_layout_destroy(h);
            }
        };

        inline void lower(const Mapping& m, Lowered& out)
        {
            const auto dyn = m.extents().dynamicValues();
            const std::string name = m.name();
            const int rc = lam_layout_create(m.schema().toString().c_str(), m.extents().toString().c_str(), dyn.data(),
                                             dyn.size(), name.c_str(), 0, 0, &out.h);
            if(rc == LAM_OK)
                return;
            if(rc == LAM_EINVAL)
                throw std::invalid_argument("copyViewB200: mapping '" + name + "' cannot be lowered to the device ("
                                            + lam_last_error() + "); use lamina::copyView for it");
            rethrow(rc);
        }

        inline const FieldAccessCount* facOf(const Mapping* m)
        {
            for(; m != nullptr; m = m->inner())
                if(auto* f = dynamic_cast<const FieldAccessCount*>(m))
                    return f;
            return nullptr;
        }

        inline const Heatmap* heatOf(const Mapping* m)
        {
            for(; m != nullptr; m = m->inner())
                if(auto* h = dynamic_cast<const Heatmap*>(m))
                    return h;
            return nullptr;
        }

        inline void split(const Mapping& m, const std::vector<std::uint64_t>& raw, std::vector<std::uint64_t>& reads,
                          std::vector<std::uint64_t>& writes, std::vector<std::vector<std::uint64_t>>& heat)
        {
            std::size_t pos = 0;
            const std::size_t L = m.schema().leafCount();
            if(facOf(&m))
            {
                reads.assign(raw.begin(), raw.begin() + L);
                writes.assign(raw.begin() + L, raw.begin() + 2 * L);
                pos = 2 * L;
            }
            if(auto* h = heatOf(&m))
                for(std::size_t nr = 0; nr < h->blobCount(); ++nr)
                {
                    heat.emplace_back(raw.begin() + pos, raw.begin() + pos + h->blockCount(nr));
                    pos += h->blockCount(nr);
                }
        }

        inline std::size_t counterWords(const Mapping& m)
        {
            std::size_t n = facOf(&m) ? 2 * m.schema().leafCount() : 0;
            if(auto* h = heatOf(&m))
                for(std::size_t nr = 0; nr < h->blobCount(); ++nr)
                    n += h->blockCount(nr);
            return n;
        }
    } // namespace b200_detail

    /// copyView(src, dst) (view.hpp:281-285, view.cpp:168-189) through the sm_100a kernels:
    /// same contract and exceptions ("incompatible views", ...); the host blobs stream through
    /// the GPU (lam_copy_host: H2D, kernel, D2H overlapped), dst blobs in/out so that bytes the
    /// copy never writes keep their values.  Counter deltas go to `deltas` when given.
    inline void copyViewB200(const View& src, View& dst, int device = 0, B200CopyCounters* deltas = nullptr)
    {
        if(!(src.schema() == dst.schema()) || !(src.extents() == dst.extents()))
            throw std::invalid_argument("incompatible views");
        b200_detail::Lowered a, b;
        b200_detail::lower(src.mapping(), a);
        b200_detail::lower(dst.mapping(), b);
        std::vector<const void*> sb;
        std::vector<void*> db;
        for(const auto& blob : src.blobs())
            sb.push_back(blob.data());
        for(auto& blob : dst.blobs())
            db.push_back(blob.data());
        std::vector<std::uint64_t> sc(b200_detail::counterWords(src.mapping()) + 1),
            dc(b200_detail::counterWords(dst.mapping()) + 1);
        const int rc = lam_copy_host(a.h, sb.data(), b.h, db.data(), device, sc.data(), dc.data());
        if(rc != LAM_OK)
            b200_detail::rethrow(rc);
        if(deltas)
        {
            *deltas = B200CopyCounters{};
            b200_detail::split(src.mapping(), sc, deltas->srcReads, deltas->srcWrites, deltas->srcHeat);
            b200_detail::split(dst.mapping(), dc, deltas->dstReads, deltas->dstWrites, deltas->dstHeat);
        }
    }
} // namespace lamina
