// Header-only C++ host mirror of the reference's hot-path API over the C ABI
// (include/lamina_b200.h).  Same names, argument meaning and exception types as
// lamina (/root/reference/proj/core/include/lamina/{layout_spec,view,instrument}.hpp),
// so reference-style host code switches by changing the namespace for the calls below:
//
//   const auto schema = lamina_b200::RecordSchema::parse(schemaText);
//   const auto ext = lamina_b200::ArrayExtents::parse("i32:[1048576]", {});
//   lamina_b200::View src(lamina_b200::parseLayout("aos-packed", schema, ext));
//   lamina_b200::View dst(lamina_b200::parseLayout("aosoa:32", schema, ext));
//   lamina_b200::copyView(src, dst);          // sm_100a kernels, stream-ordered
//
// Not mirrored: user-defined Mapping subclasses (mapping.hpp:44-155) -- a device view needs a
// mapping the layout grammar can name; RecordSchema / ArrayExtents here are validated,
// canonical text (no leaf-table or coordinate API).  Views the reference already owns go
// through lamina::copyViewB200 (include/lamina_b200_binding.hpp).
//
// Errors are rethrown as std::invalid_argument / std::out_of_range / std::overflow_error /
// std::logic_error with the reference's messages; CUDA failures as std::runtime_error.
#pragma once

#include "lamina_b200.h"

#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace lamina_b200
{
    inline void check(int rc)
    {
        if(rc == LAM_OK)
            return;
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

    /// lamina::MappingPtr equivalent: a lowered mapping (schema + extents + layout).
    class Mapping
    {
    public:
        Mapping(const std::string& schema, const std::string& extents, const std::string& layout,
                const std::vector<std::uint64_t>& dyn = {}, int wrap = 0, std::uint64_t granularity = 0)
        {
            lam_layout* h = nullptr;
            check(lam_layout_create(schema.c_str(), extents.c_str(), dyn.data(), dyn.size(), layout.c_str(), wrap,
                                    granularity, &h));
            h_.reset(h, lam_layout_destroy);
        }

        std::string name() const
        {
            std::string s(lam_layout_name(h_.get(), nullptr, 0), '\0');
            lam_layout_name(h_.get(), s.data(), s.size() + 1);
            return s;
        }
        std::size_t blobCount() const
        {
            return lam_layout_blob_count(h_.get());
        }
        std::uint64_t blobSize(std::size_t nr) const
        {
            return lam_layout_blob_size(h_.get(), nr);
        }
        std::uint64_t elementCount() const
        {
            return lam_layout_element_count(h_.get());
        }
        const lam_layout* handle() const
        {
            return h_.get();
        }

        /// Mapping::contiguousRun (mapping.hpp:122-135): (nr, offset) when the n values of the
        /// leaf starting at `linear` are contiguous; nullopt otherwise.
        std::optional<std::pair<std::size_t, std::uint64_t>> contiguousRun(std::uint64_t linear, std::size_t flatLeaf,
                                                                           std::uint64_t n) const
        {
            int has = 0;
            std::size_t nr = 0;
            std::uint64_t off = 0;
            check(lam_layout_contiguous_run(h_.get(), linear, flatLeaf, n, &has, &nr, &off));
            if(!has)
                return std::nullopt;
            return std::make_pair(nr, off);
        }

        /// the .meta sidecar writeViewDump writes for a view of this mapping (view_io.cpp:30-44)
        std::string dumpMeta() const
        {
            std::string s(lam_layout_dump_meta(h_.get(), nullptr, 0), '\0');
            lam_layout_dump_meta(h_.get(), s.data(), s.size() + 1);
            return s;
        }

        /// adopt a layout handle created by the C ABI (lam_view_restore)
        static std::shared_ptr<const Mapping> adopt(lam_layout* h)
        {
            auto m = std::shared_ptr<Mapping>(new Mapping());
            m->h_.reset(h, lam_layout_destroy);
            return m;
        }

    private:
        Mapping() = default;
        std::shared_ptr<lam_layout> h_;
    };

    using MappingPtr = std::shared_ptr<const Mapping>;

    /// lamina::RecordSchema::parse (record.cpp:364-479): validated, held as canonical text.
    class RecordSchema
    {
    public:
        static RecordSchema parse(const std::string& text)
        {
            lam_layout* h = nullptr;
            check(lam_layout_create(text.c_str(), "i32:[1]", nullptr, 0, "aos-packed", 0, 0, &h));
            RecordSchema s;
            s.text_.resize(lam_layout_schema(h, nullptr, 0));
            lam_layout_schema(h, s.text_.data(), s.text_.size() + 1);
            lam_layout_destroy(h);
            return s;
        }
        const std::string& toString() const noexcept
        {
            return text_;
        }
        bool operator==(const RecordSchema& o) const noexcept
        {
            return text_ == o.text_;
        }

    private:
        std::string text_;
    };

    /// lamina::ArrayExtents::parse(text, dynamicValues) (extents.cpp:118-177): validated
    /// ("index type overflow", ...), canonical text plus the dynamic values.
    class ArrayExtents
    {
    public:
        static ArrayExtents parse(const std::string& text, const std::vector<std::uint64_t>& dynamicValues)
        {
            lam_layout* h = nullptr;
            check(lam_layout_create("Record{v:u8}", text.c_str(), dynamicValues.data(), dynamicValues.size(),
                                    "aos-packed", 0, 0, &h));
            ArrayExtents e;
            e.text_.resize(lam_layout_extents(h, nullptr, 0));
            lam_layout_extents(h, e.text_.data(), e.text_.size() + 1);
            e.count_ = lam_layout_element_count(h);
            lam_layout_destroy(h);
            e.dyn_ = dynamicValues;
            return e;
        }
        const std::string& toString() const noexcept
        {
            return text_;
        }
        const std::vector<std::uint64_t>& dynamicValues() const noexcept
        {
            return dyn_;
        }
        bool isFullyStatic() const noexcept
        {
            return dyn_.empty();
        }
        std::uint64_t elementCount() const noexcept
        {
            return count_;
        }

    private:
        std::string text_;
        std::vector<std::uint64_t> dyn_;
        std::uint64_t count_ = 0;
    };

    /// lamina::parseLayout(text, schema, extents) (layout_spec.hpp:19), schema/extents as text.
    inline MappingPtr parseLayout(const std::string& text, const std::string& schema, const std::string& extents,
                                  const std::vector<std::uint64_t>& dyn = {})
    {
        return std::make_shared<const Mapping>(schema, extents, text, dyn);
    }

    /// lamina::parseLayout(std::string_view, const RecordSchema&, const ArrayExtents&)
    /// (layout_spec.hpp:19), the reference's own signature.
    inline MappingPtr parseLayout(const std::string& text, const RecordSchema& schema, const ArrayExtents& extents)
    {
        return std::make_shared<const Mapping>(schema.toString(), extents.toString(), text, extents.dynamicValues());
    }

    /// lamina::View on a device: zero-filled blobs in HBM (or adopted device pointers).
    class View
    {
    public:
        explicit View(MappingPtr m, int device = 0, void* stream = nullptr) : m_(std::move(m))
        {
            lam_view* v = nullptr;
            check(lam_view_alloc(m_->handle(), device, stream, &v));
            v_.reset(v, lam_view_free);
        }
        /// View(MappingPtr, std::vector<Blob>) (view.cpp:105-118): adopts device blobs of the
        /// given sizes ("blob count mismatch" / "blob size mismatch" as the reference).
        View(MappingPtr m, const std::vector<void*>& deviceBlobs, const std::vector<uint64_t>& blobBytes,
             int device = 0)
            : m_(std::move(m))
        {
            if(blobBytes.size() != deviceBlobs.size())
                throw std::invalid_argument("blob count mismatch: " + std::to_string(deviceBlobs.size())
                                            + " blobs, " + std::to_string(blobBytes.size()) + " sizes");
            lam_view* v = nullptr;
            check(lam_view_wrap(m_->handle(), device, deviceBlobs.data(), blobBytes.data(), deviceBlobs.size(), &v));
            v_.reset(v, lam_view_free);
        }
        const Mapping& mapping() const
        {
            return *m_;
        }
        void* blob(std::size_t nr) const
        {
            return lam_view_blob(v_.get(), nr);
        }
        lam_view* handle() const
        {
            return v_.get();
        }
        /// View::isTriviallyRelocatable / blobBytes / stateBytes (view.cpp:145-162)
        bool isTriviallyRelocatable() const noexcept
        {
            return lam_view_is_trivially_relocatable(v_.get()) != 0;
        }
        std::size_t blobBytes() const noexcept
        {
            return static_cast<std::size_t>(lam_view_blob_bytes(v_.get()));
        }
        std::size_t stateBytes() const noexcept
        {
            return static_cast<std::size_t>(lam_view_state_bytes(v_.get()));
        }

        /// FieldAccessCount::counters() of an instrumented view: (reads, writes) per leaf
        std::pair<std::vector<std::uint64_t>, std::vector<std::uint64_t>> counters(std::size_t leaves) const
        {
            std::vector<std::uint64_t> r(leaves), w(leaves);
            check(lam_counters_read(v_.get(), r.data(), w.data()));
            return {r, w};
        }

        /// adopt a (layout, view) pair created by the C ABI (lam_view_restore)
        View(MappingPtr m, lam_view* v) : m_(std::move(m))
        {
            v_.reset(v, lam_view_free);
        }

    private:
        MappingPtr m_;
        std::shared_ptr<lam_view> v_;
    };

    /// lamina::writeViewDump (view_io.cpp:28-59): <stem>.meta + <stem>.blob<nr>.bin
    inline void writeViewDump(const View& view, const std::string& stem)
    {
        check(lam_view_dump(view.handle(), stem.c_str()));
    }

    /// lamina::readViewDump (view_io.cpp:61-129) onto a device
    inline View readViewDump(const std::string& stem, int device = 0, void* stream = nullptr)
    {
        lam_layout* l = nullptr;
        lam_view* v = nullptr;
        check(lam_view_restore(stem.c_str(), device, stream, &l, &v));
        return View(Mapping::adopt(l), v);
    }

    /// lamina::copyView(const View&, View&) (view.hpp:285) on the GPU, stream-ordered.
    inline void copyView(const View& src, View& dst, void* stream = nullptr)
    {
        check(lam_copy(src.handle(), dst.handle(), stream));
    }

    /// copyView over host blobs (dst blobs in/out), streamed through the GPU.
    inline void copyViewHost(const Mapping& src, const std::vector<const void*>& srcBlobs, const Mapping& dst,
                             const std::vector<void*>& dstBlobs, int device = 0)
    {
        check(lam_copy_host(src.handle(), srcBlobs.data(), dst.handle(), dstBlobs.data(), device, nullptr, nullptr));
    }
} // namespace lamina_b200
