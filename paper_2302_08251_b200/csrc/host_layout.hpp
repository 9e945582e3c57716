// Host side of the boundary: record schemas, array extents, the layout grammar and
// the mapping tree, lowered into the device plan (lam_plan.h).
//
// Mirrors the reference's runtime-typed API (record.hpp, extents.hpp, mapping.hpp,
// mappings.hpp, computed.hpp, instrument.hpp, layout_spec.hpp under
// /root/reference/proj/core/include/lamina) with the same names, validation rules and
// exception messages, so that errors surface exactly where the reference raises them.
#pragma once

#include "lam_plan.h"

#include <algorithm>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace lamb
{
    // ---- scalars (scalar.hpp:16-70) -----------------------------------------------------
    enum Scalar : uint8_t
    {
        I8,
        I16,
        I32,
        I64,
        U8,
        U16,
        U32,
        U64,
        F32,
        F64,
        Bool
    };

    size_t scalarSize(int s);
    bool isSignedInt(int s);
    bool isUnsignedInt(int s);
    inline bool isInteger(int s)
    {
        return isSignedInt(s) || isUnsignedInt(s);
    }
    inline bool isFloat(int s)
    {
        return s == F32 || s == F64;
    }
    const char* scalarName(int s);
    int parseScalar(std::string_view text); // throws invalid_argument
    bool convertible(int from, int to);     // ScalarValue::convertible, scalar.hpp:308-319

    // ---- record schema (record.hpp:84-248) ---------------------------------------------
    struct SNode;
    using SNodePtr = std::shared_ptr<const SNode>;
    struct SNode
    {
        enum Kind
        {
            Record,
            Array,
            Leaf
        } kind = Leaf;
        int scalar = F64;
        uint64_t count = 0;
        SNodePtr element;
        std::vector<std::pair<std::string, SNodePtr>> fields;
        size_t childCount() const;
        SNodePtr child(size_t i) const;
    };

    struct LeafDesc
    {
        std::vector<uint32_t> coord;
        std::string path;
        int type = F64;
        size_t size = 0;
        size_t offsetPacked = 0;
        size_t offsetAligned = 0;
    };

    class Schema
    {
    public:
        explicit Schema(SNodePtr root);
        static Schema parse(std::string_view text);
        static SNodePtr leaf(int s);
        static SNodePtr record(std::vector<std::pair<std::string, SNodePtr>> fields);
        static SNodePtr array(uint64_t count, SNodePtr element);

        const SNodePtr& root() const
        {
            return root_;
        }
        size_t leafCount() const
        {
            return leaves_.size();
        }
        const LeafDesc& leaf(size_t f) const
        {
            return leaves_.at(f);
        }
        const std::vector<LeafDesc>& leaves() const
        {
            return leaves_;
        }
        size_t sizePacked() const
        {
            return sizePacked_;
        }
        size_t sizeAligned() const
        {
            return sizeAligned_;
        }
        SNodePtr nodeAt(const std::vector<uint32_t>& coord) const;
        std::vector<uint32_t> coordOf(std::string_view dotted) const;
        std::string pathOf(const std::vector<uint32_t>& coord) const;
        std::pair<size_t, size_t> leafRange(const std::vector<uint32_t>& coord) const;
        std::string toString() const;
        bool operator==(const Schema& o) const;

    private:
        SNodePtr root_;
        std::vector<LeafDesc> leaves_;
        size_t sizePacked_ = 0;
        size_t sizeAligned_ = 0;
    };

    // ---- array extents (extents.hpp:14-165) ---------------------------------------------
    enum IndexType : uint8_t
    {
        IT_I16,
        IT_I32,
        IT_I64,
        IT_U16,
        IT_U32,
        IT_U64
    };
    constexpr uint64_t kDyn = ~uint64_t{0};

    class Extents
    {
    public:
        Extents(IndexType it, std::vector<uint64_t> dims, std::vector<uint64_t> dynValues);
        static Extents parse(std::string_view text, const uint64_t* dyn, size_t ndyn);
        uint64_t elementCount() const
        {
            return n_;
        }
        IndexType indexType() const
        {
            return it_;
        }
        bool isFullyStatic() const
        {
            return dynValues_.empty();
        }
        size_t runtimeStateBytes() const;
        std::string toString() const;
        const std::vector<uint64_t>& dynamicValues() const
        {
            return dynValues_;
        }
        bool operator==(const Extents& o) const
        {
            return it_ == o.it_ && dims_ == o.dims_ && dynValues_ == o.dynValues_;
        }

    private:
        IndexType it_;
        std::vector<uint64_t> dims_;
        std::vector<uint64_t> dynValues_;
        uint64_t n_ = 1;
    };

    // ---- plan builder -------------------------------------------------------------------
    struct PlanBuilder
    {
        std::vector<lamp_node> nodes;
        std::vector<lamp_stream> streams;
        // one byte bitmap per PHYS stream for the hole analysis
        std::vector<std::vector<uint8_t>> coverage;
        uint16_t addNode(const lamp_node& n);
        uint16_t physStream(uint32_t nr, uint64_t base, uint64_t bs, uint64_t lanes, uint64_t& inblock);
        uint16_t bitsStream(uint32_t nr, uint32_t bits);
        void markCoverage(uint16_t stream, uint64_t inblock, uint64_t laneStride, uint64_t size);
        void finalize();
    };

    // ---- mappings (mapping.hpp:44-155) -------------------------------------------------
    class Map;
    using MapPtr = std::shared_ptr<const Map>;
    using Factory = std::function<MapPtr(Schema, Extents)>;

    class Map
    {
    public:
        Map(Schema s, Extents e) : schema_(std::move(s)), extents_(std::move(e))
        {
        }
        virtual ~Map() = default;
        const Schema& schema() const
        {
            return schema_;
        }
        const Extents& extents() const
        {
            return extents_;
        }
        uint64_t elementCount() const
        {
            return extents_.elementCount();
        }
        virtual std::string name() const = 0;
        virtual size_t blobCount() const = 0;
        virtual uint64_t blobSize(size_t nr) const = 0;
        virtual bool isComputed(size_t) const
        {
            return false;
        }
        bool isFullyPhysical() const;
        virtual bool hasMutableState() const
        {
            return false;
        }
        // Mapping::runtimeStateBytes (mapping.hpp:145-148): dynamic extents' slots, plus inner
        // mappings' and counters' bytes in the wrappers (computed.cpp:396-399,499-502,
        // mappings.cpp:386-389, instrument.cpp:79-82,197-200)
        virtual size_t runtimeStateBytes() const
        {
            return extents_.runtimeStateBytes();
        }
        // physicalOffset without bounds checks; throws logic_error for computed leaves
        virtual std::pair<size_t, uint64_t> offsetOf(uint64_t i, size_t f) const;
        // lower leaf f into plan nodes; blob numbers shifted by `blobShift`
        virtual uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const = 0;
        virtual const Map* inner() const
        {
            return nullptr;
        }
        // deepest node chain produced by lower(), for the device recursion bound
        virtual int depth() const
        {
            return 1;
        }

    protected:
        Schema schema_;
        Extents extents_;
    };

    class AoSMap final : public Map
    {
    public:
        AoSMap(Schema s, Extents e, bool aligned);
        std::string name() const override
        {
            return aligned_ ? "aos-aligned" : "aos-packed";
        }
        size_t blobCount() const override
        {
            return 1;
        }
        uint64_t blobSize(size_t) const override
        {
            return elementCount() * recordSize_;
        }
        std::pair<size_t, uint64_t> offsetOf(uint64_t i, size_t f) const override
        {
            return {0, i * recordSize_ + leafOffset_[f]};
        }
        uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const override;

    private:
        bool aligned_;
        uint64_t recordSize_;
        std::vector<uint64_t> leafOffset_;
    };

    class SoAMap final : public Map
    {
    public:
        SoAMap(Schema s, Extents e, bool multiBlob);
        std::string name() const override
        {
            return multi_ ? "soa-mb" : "soa-sb";
        }
        size_t blobCount() const override
        {
            return multi_ ? schema_.leafCount() : 1;
        }
        uint64_t blobSize(size_t nr) const override;
        std::pair<size_t, uint64_t> offsetOf(uint64_t i, size_t f) const override;
        uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const override;

    private:
        bool multi_;
        std::vector<uint64_t> subarrayBase_;
    };

    class AoSoAMap final : public Map
    {
    public:
        AoSoAMap(Schema s, Extents e, uint64_t lanes);
        std::string name() const override
        {
            return "aosoa:" + std::to_string(lanes_);
        }
        size_t blobCount() const override
        {
            return 1;
        }
        uint64_t blobSize(size_t) const override;
        std::pair<size_t, uint64_t> offsetOf(uint64_t i, size_t f) const override;
        uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const override;

    private:
        uint64_t lanes_;
        uint64_t blockSize_;
    };

    class OneMap final : public Map
    {
    public:
        OneMap(Schema s, Extents e);
        std::string name() const override
        {
            return "one";
        }
        size_t blobCount() const override
        {
            return 1;
        }
        uint64_t blobSize(size_t) const override
        {
            return schema_.sizePacked();
        }
        std::pair<size_t, uint64_t> offsetOf(uint64_t, size_t f) const override
        {
            return {0, schema_.leaf(f).offsetPacked};
        }
        uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const override;
    };

    class SplitMap final : public Map
    {
    public:
        SplitMap(Schema s, Extents e, std::vector<std::vector<uint32_t>> selectors, const Factory& a,
                 const Factory& b);
        std::string name() const override;
        size_t blobCount() const override
        {
            return a_->blobCount() + b_->blobCount();
        }
        uint64_t blobSize(size_t nr) const override
        {
            return nr < a_->blobCount() ? a_->blobSize(nr) : b_->blobSize(nr - a_->blobCount());
        }
        bool isComputed(size_t f) const override;
        bool hasMutableState() const override
        {
            return a_->hasMutableState() || b_->hasMutableState();
        }
        size_t runtimeStateBytes() const override
        {
            return extents_.runtimeStateBytes() + a_->runtimeStateBytes() + b_->runtimeStateBytes();
        }
        std::pair<size_t, uint64_t> offsetOf(uint64_t i, size_t f) const override;
        uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const override;
        int depth() const override
        {
            return std::max(a_->depth(), b_->depth());
        }

    private:
        std::vector<std::vector<uint32_t>> selectors_;
        MapPtr a_, b_;
        std::vector<std::pair<bool, size_t>> route_;
    };

    class NullMap final : public Map
    {
    public:
        NullMap(Schema s, Extents e) : Map(std::move(s), std::move(e))
        {
        }
        std::string name() const override
        {
            return "null";
        }
        size_t blobCount() const override
        {
            return 0;
        }
        uint64_t blobSize(size_t) const override
        {
            return 0;
        }
        bool isComputed(size_t) const override
        {
            return true;
        }
        uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const override;
    };

    class BitpackIntMap final : public Map
    {
    public:
        BitpackIntMap(Schema s, Extents e, std::vector<unsigned> bits);
        std::string name() const override;
        size_t blobCount() const override
        {
            return bits_.size();
        }
        uint64_t blobSize(size_t nr) const override;
        bool isComputed(size_t) const override
        {
            return true;
        }
        uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const override;

    private:
        std::vector<unsigned> bits_;
    };

    class BitpackFloatMap final : public Map
    {
    public:
        BitpackFloatMap(Schema s, Extents e, std::vector<std::pair<unsigned, unsigned>> em);
        std::string name() const override;
        size_t blobCount() const override
        {
            return em_.size();
        }
        uint64_t blobSize(size_t nr) const override;
        bool isComputed(size_t) const override
        {
            return true;
        }
        uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const override;

    private:
        std::vector<std::pair<unsigned, unsigned>> em_;
    };

    struct TypeChange
    {
        bool byType = true;
        int type = F64;                // selector type
        std::vector<uint32_t> coord;   // selector coord
        int target = F32;
    };

    class ChangeTypeMap final : public Map
    {
    public:
        ChangeTypeMap(Schema s, Extents e, std::vector<TypeChange> changes, const Factory& inner);
        std::string name() const override;
        size_t blobCount() const override
        {
            return inner_->blobCount();
        }
        uint64_t blobSize(size_t nr) const override
        {
            return inner_->blobSize(nr);
        }
        bool isComputed(size_t f) const override
        {
            return storage_[f] != schema_.leaf(f).type || inner_->isComputed(f);
        }
        bool hasMutableState() const override
        {
            return inner_->hasMutableState();
        }
        size_t runtimeStateBytes() const override
        {
            return extents_.runtimeStateBytes() + inner_->runtimeStateBytes();
        }
        std::pair<size_t, uint64_t> offsetOf(uint64_t i, size_t f) const override;
        uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const override;
        const Map* inner() const override
        {
            return inner_.get();
        }
        int depth() const override
        {
            return 1 + inner_->depth();
        }

    private:
        std::vector<TypeChange> changes_;
        std::vector<int> storage_;
        MapPtr inner_;
    };

    class BytesplitMap final : public Map
    {
    public:
        BytesplitMap(Schema s, Extents e, const Factory& inner);
        std::string name() const override
        {
            return "bytesplit:" + inner_->name();
        }
        size_t blobCount() const override
        {
            return inner_->blobCount();
        }
        uint64_t blobSize(size_t nr) const override
        {
            return inner_->blobSize(nr);
        }
        bool isComputed(size_t) const override
        {
            return true;
        }
        bool hasMutableState() const override
        {
            return inner_->hasMutableState();
        }
        size_t runtimeStateBytes() const override
        {
            return extents_.runtimeStateBytes() + inner_->runtimeStateBytes();
        }
        uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const override;
        const Map* inner() const override
        {
            return inner_.get();
        }
        int depth() const override
        {
            return 1 + inner_->depth();
        }

    private:
        MapPtr inner_;
    };

    // Instrumentation wrappers (instrument.hpp:27-127): counters live on the device view.
    class FieldAccessCountMap final : public Map
    {
    public:
        explicit FieldAccessCountMap(MapPtr inner);
        std::string name() const override
        {
            return "field-access-count(" + inner_->name() + ")";
        }
        size_t runtimeStateBytes() const override
        {
            return extents_.runtimeStateBytes() + inner_->runtimeStateBytes() + 2 * schema_.leafCount() * 8;
        }
        size_t blobCount() const override
        {
            return inner_->blobCount();
        }
        uint64_t blobSize(size_t nr) const override
        {
            return inner_->blobSize(nr);
        }
        bool isComputed(size_t f) const override
        {
            return inner_->isComputed(f);
        }
        bool hasMutableState() const override
        {
            return true;
        }
        std::pair<size_t, uint64_t> offsetOf(uint64_t i, size_t f) const override
        {
            return inner_->offsetOf(i, f);
        }
        uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const override
        {
            return inner_->lower(f, blobShift, pb);
        }
        const Map* inner() const override
        {
            return inner_.get();
        }
        int depth() const override
        {
            return inner_->depth();
        }

    private:
        MapPtr inner_;
    };

    class HeatmapMap final : public Map
    {
    public:
        HeatmapMap(MapPtr inner, uint64_t granularity);
        std::string name() const override
        {
            return "heatmap:" + std::to_string(gran_) + "(" + inner_->name() + ")";
        }
        size_t runtimeStateBytes() const override
        {
            size_t blocks = 0;
            for(size_t nr = 0; nr < blobCount(); ++nr)
                blocks += blockCount(nr);
            return extents_.runtimeStateBytes() + inner_->runtimeStateBytes() + blocks * 8;
        }
        size_t blobCount() const override
        {
            return inner_->blobCount();
        }
        uint64_t blobSize(size_t nr) const override
        {
            return inner_->blobSize(nr);
        }
        bool isComputed(size_t f) const override
        {
            return inner_->isComputed(f);
        }
        bool hasMutableState() const override
        {
            return true;
        }
        std::pair<size_t, uint64_t> offsetOf(uint64_t i, size_t f) const override
        {
            return inner_->offsetOf(i, f);
        }
        uint16_t lower(size_t f, uint32_t blobShift, PlanBuilder& pb) const override
        {
            return inner_->lower(f, blobShift, pb);
        }
        const Map* inner() const override
        {
            return inner_.get();
        }
        int depth() const override
        {
            return inner_->depth();
        }
        uint64_t granularity() const
        {
            return gran_;
        }
        uint64_t blockCount(size_t nr) const
        {
            return (blobSize(nr) + gran_ - 1) / gran_;
        }

    private:
        MapPtr inner_;
        uint64_t gran_;
    };

    // layout grammar (layout_spec.cpp:37-167) + wrapper names
    MapPtr parseLayout(std::string_view text, const Schema& schema, const Extents& extents);

    // Fully lowered layout: what a lam_layout handle owns.
    struct Lowered
    {
        MapPtr map;
        std::vector<uint16_t> roots;
        std::vector<lamp_node> nodes;
        std::vector<lamp_stream> streams;
        bool fac = false;
        bool heat = false;
        uint64_t heatGran = 0;
        std::vector<uint64_t> heatOffset; // per blob
        uint64_t heatTotal = 0;
        uint64_t shardUnit = 1; // elements
        bool int32Index = true;
    };

    std::shared_ptr<Lowered> lower(MapPtr map);

    const FieldAccessCountMap* findFac(const Map* m);
    const HeatmapMap* findHeat(const Map* m);
} // namespace lamb
