// Host-side schema / extents / layout grammar and the lowering of mapping trees into
// device plans.  See host_layout.hpp.  Semantics follow the reference file:line cited
// at each function; the code is written against the plan representation, not ported.
#include "host_layout.hpp"

#include <algorithm>
#include <cctype>
#include <functional>
#include <numeric>
#include <unordered_set>

namespace lamb
{
    // ======================================================================================
    // scalars — scalar.hpp:16-70, scalar.cpp:8-58
    // ======================================================================================
    size_t scalarSize(int s)
    {
        switch(s)
        {
        case I8:
        case U8:
        case Bool:
            return 1;
        case I16:
        case U16:
            return 2;
        case I32:
        case U32:
        case F32:
            return 4;
        default:
            return 8;
        }
    }
    bool isSignedInt(int s)
    {
        return s == I8 || s == I16 || s == I32 || s == I64;
    }
    bool isUnsignedInt(int s)
    {
        return s == U8 || s == U16 || s == U32 || s == U64;
    }
    static const char* const kScalarNames[] = {"i8", "i16", "i32", "i64", "u8", "u16", "u32", "u64", "f32", "f64", "bool"};
    const char* scalarName(int s)
    {
        return (s >= 0 && s <= Bool) ? kScalarNames[s] : "?";
    }
    int parseScalar(std::string_view text)
    {
        for(int s = 0; s <= Bool; ++s)
            if(text == kScalarNames[s])
                return s;
        throw std::invalid_argument("unknown scalar type: '" + std::string(text) + "'");
    }
    bool convertible(int from, int to)
    {
        return from == to || (isFloat(from) && isFloat(to)) || (isSignedInt(from) && isSignedInt(to))
            || (isUnsignedInt(from) && isUnsignedInt(to));
    }

    // ======================================================================================
    // schema — record.hpp:84-248, record.cpp:86-158 (leaf table), 364-479 (grammar)
    // ======================================================================================
    size_t SNode::childCount() const
    {
        return kind == Record ? fields.size() : kind == Array ? static_cast<size_t>(count) : 0;
    }
    SNodePtr SNode::child(size_t i) const
    {
        if(kind == Record)
            return fields.at(i).second;
        if(kind == Array && i < count)
            return element;
        throw std::out_of_range("record child index out of range");
    }

    static bool validTag(const std::string& t)
    {
        if(t.empty() || std::isdigit(static_cast<unsigned char>(t[0])))
            return false;
        for(char c : t)
            if(!(std::isalnum(static_cast<unsigned char>(c)) || c == '_'))
                return false;
        return true;
    }

    SNodePtr Schema::leaf(int s)
    {
        auto n = std::make_shared<SNode>();
        n->kind = SNode::Leaf;
        n->scalar = s;
        return n;
    }
    SNodePtr Schema::record(std::vector<std::pair<std::string, SNodePtr>> fields)
    {
        auto n = std::make_shared<SNode>();
        n->kind = SNode::Record;
        std::unordered_set<std::string> seen;
        for(auto& f : fields)
        {
            if(!validTag(f.first))
                throw std::invalid_argument("invalid field tag: '" + f.first + "'");
            if(!seen.insert(f.first).second)
                throw std::invalid_argument("duplicate field tag: '" + f.first + "'");
        }
        n->fields = std::move(fields);
        return n;
    }
    SNodePtr Schema::array(uint64_t count, SNodePtr element)
    {
        if(count < 1)
            throw std::invalid_argument("fixed array count must be >= 1");
        auto n = std::make_shared<SNode>();
        n->kind = SNode::Array;
        n->count = count;
        n->element = std::move(element);
        return n;
    }

    Schema::Schema(SNodePtr root) : root_(std::move(root))
    {
        // DFS pre-order leaf table with packed and naturally aligned offsets
        std::vector<uint32_t> coord;
        std::string path;
        std::function<void(const SNodePtr&)> walk = [&](const SNodePtr& n)
        {
            if(n->kind == SNode::Leaf)
            {
                LeafDesc d;
                d.coord = coord;
                d.path = path;
                d.type = n->scalar;
                d.size = scalarSize(n->scalar);
                leaves_.push_back(std::move(d));
                return;
            }
            for(size_t i = 0; i < n->childCount(); ++i)
            {
                const size_t keep = path.size();
                if(n->kind == SNode::Record)
                {
                    if(!path.empty())
                        path += '.';
                    path += n->fields[i].first;
                }
                else
                    path += "[" + std::to_string(i) + "]";
                coord.push_back(static_cast<uint32_t>(i));
                walk(n->child(i));
                coord.pop_back();
                path.resize(keep);
            }
        };
        walk(root_);
        size_t packed = 0, aligned = 0, maxAlign = 1;
        for(auto& d : leaves_)
        {
            d.offsetPacked = packed;
            packed += d.size;
            aligned = (aligned + d.size - 1) / d.size * d.size;
            d.offsetAligned = aligned;
            aligned += d.size;
            maxAlign = std::max(maxAlign, d.size);
        }
        sizePacked_ = packed;
        sizeAligned_ = (aligned + maxAlign - 1) / maxAlign * maxAlign;
    }

    namespace
    {
        struct SchemaText
        {
            std::string_view t;
            size_t p = 0;
            [[noreturn]] void fail(const std::string& what)
            {
                throw std::invalid_argument("schema parse error at position " + std::to_string(p) + ": " + what);
            }
            void ws()
            {
                while(p < t.size() && std::isspace(static_cast<unsigned char>(t[p])))
                    ++p;
            }
            char peek()
            {
                ws();
                return p < t.size() ? t[p] : '\0';
            }
            void expect(char c)
            {
                if(peek() != c)
                    fail(std::string("expected '") + c + "'");
                ++p;
            }
            std::string word()
            {
                ws();
                size_t s = p;
                while(p < t.size() && (std::isalnum(static_cast<unsigned char>(t[p])) || t[p] == '_'))
                    ++p;
                if(s == p)
                    fail("expected identifier");
                return std::string(t.substr(s, p - s));
            }
            uint64_t number()
            {
                ws();
                size_t s = p;
                while(p < t.size() && std::isdigit(static_cast<unsigned char>(t[p])))
                    ++p;
                if(s == p)
                    fail("expected number");
                return std::stoull(std::string(t.substr(s, p - s)));
            }
            SNodePtr node()
            {
                SNodePtr base;
                const std::string w = word();
                if(w == "Record")
                {
                    expect('{');
                    std::vector<std::pair<std::string, SNodePtr>> fields;
                    if(peek() != '}')
                    {
                        while(true)
                        {
                            std::string tag = word();
                            expect(':');
                            fields.emplace_back(std::move(tag), node());
                            if(peek() == ',')
                            {
                                ++p;
                                continue;
                            }
                            break;
                        }
                    }
                    expect('}');
                    base = Schema::record(std::move(fields));
                }
                else
                    base = Schema::leaf(parseScalar(w));
                std::vector<uint64_t> counts;
                while(peek() == '[')
                {
                    ++p;
                    counts.push_back(number());
                    expect(']');
                }
                // T[a][b] is a elements of T[b]
                for(auto it = counts.rbegin(); it != counts.rend(); ++it)
                    base = Schema::array(*it, base);
                return base;
            }
        };

        void printNode(std::string& out, const SNodePtr& n)
        {
            if(n->kind == SNode::Leaf)
                out += scalarName(n->scalar);
            else if(n->kind == SNode::Record)
            {
                out += "Record{";
                for(size_t i = 0; i < n->fields.size(); ++i)
                {
                    if(i)
                        out += ',';
                    out += n->fields[i].first + ":";
                    printNode(out, n->fields[i].second);
                }
                out += '}';
            }
            else
            {
                std::vector<uint64_t> counts;
                SNodePtr in = n;
                while(in->kind == SNode::Array)
                {
                    counts.push_back(in->count);
                    in = in->element;
                }
                printNode(out, in);
                for(auto c : counts)
                    out += "[" + std::to_string(c) + "]";
            }
        }

        bool sameTree(const SNodePtr& a, const SNodePtr& b)
        {
            if(a == b)
                return true;
            if(!a || !b || a->kind != b->kind)
                return false;
            if(a->kind == SNode::Leaf)
                return a->scalar == b->scalar;
            if(a->kind == SNode::Array)
                return a->count == b->count && sameTree(a->element, b->element);
            if(a->fields.size() != b->fields.size())
                return false;
            for(size_t i = 0; i < a->fields.size(); ++i)
                if(a->fields[i].first != b->fields[i].first || !sameTree(a->fields[i].second, b->fields[i].second))
                    return false;
            return true;
        }
    } // namespace

    Schema Schema::parse(std::string_view text)
    {
        SchemaText st{text};
        SNodePtr root = st.node();
        st.ws();
        if(st.p != text.size())
            st.fail("trailing characters");
        return Schema(root);
    }

    std::string Schema::toString() const
    {
        std::string out;
        printNode(out, root_);
        return out;
    }

    bool Schema::operator==(const Schema& o) const
    {
        return sameTree(root_, o.root_);
    }

    SNodePtr Schema::nodeAt(const std::vector<uint32_t>& coord) const
    {
        SNodePtr n = root_;
        for(auto i : coord)
        {
            if(!n || i >= n->childCount())
                return nullptr;
            n = n->child(i);
        }
        return n;
    }

    // record.cpp:220-277
    std::vector<uint32_t> Schema::coordOf(std::string_view dotted) const
    {
        std::vector<uint32_t> path;
        SNodePtr n = root_;
        auto descend = [&](std::string_view seg)
        {
            if(!n)
                throw std::invalid_argument("no such field: '" + std::string(seg) + "'");
            if(!seg.empty() && std::isdigit(static_cast<unsigned char>(seg[0])))
            {
                const auto idx = static_cast<uint32_t>(std::stoul(std::string(seg)));
                if(idx >= n->childCount())
                    throw std::invalid_argument("no such field: index " + std::string(seg));
                path.push_back(idx);
                n = n->child(idx);
                return;
            }
            if(n->kind != SNode::Record)
                throw std::invalid_argument("no such field: '" + std::string(seg) + "'");
            for(size_t i = 0; i < n->fields.size(); ++i)
                if(n->fields[i].first == seg)
                {
                    path.push_back(static_cast<uint32_t>(i));
                    n = n->fields[i].second;
                    return;
                }
            throw std::invalid_argument("no such field: '" + std::string(seg) + "'");
        };
        size_t pos = 0;
        while(pos < dotted.size())
        {
            const size_t nx = dotted.find_first_of(".[", pos);
            if(nx == std::string_view::npos)
            {
                descend(dotted.substr(pos));
                break;
            }
            if(nx > pos)
                descend(dotted.substr(pos, nx - pos));
            if(dotted[nx] == '.')
            {
                pos = nx + 1;
                continue;
            }
            const size_t close = dotted.find(']', nx);
            if(close == std::string_view::npos)
                throw std::invalid_argument("no such field: unbalanced '[' in path");
            descend(dotted.substr(nx + 1, close - nx - 1));
            pos = close + 1;
            if(pos < dotted.size() && dotted[pos] == '.')
                ++pos;
        }
        return path;
    }

    std::string Schema::pathOf(const std::vector<uint32_t>& coord) const
    {
        std::string out;
        SNodePtr n = root_;
        for(auto i : coord)
        {
            if(!n || i >= n->childCount())
                throw std::invalid_argument("no such field: coordinate");
            if(n->kind == SNode::Record)
            {
                if(!out.empty())
                    out += '.';
                out += n->fields[i].first;
            }
            else
                out += "[" + std::to_string(i) + "]";
            n = n->child(i);
        }
        return out;
    }

    static bool isPrefix(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b)
    {
        return a.size() <= b.size() && std::equal(a.begin(), a.end(), b.begin());
    }

    std::pair<size_t, size_t> Schema::leafRange(const std::vector<uint32_t>& coord) const
    {
        if(!nodeAt(coord))
            throw std::invalid_argument("no such field: coordinate");
        size_t first = leaves_.size(), last = leaves_.size();
        for(size_t i = 0; i < leaves_.size(); ++i)
            if(isPrefix(coord, leaves_[i].coord))
            {
                if(first == leaves_.size())
                    first = i;
                last = i + 1;
            }
        if(first == leaves_.size())
            first = last = 0;
        return {first, last};
    }

    // ======================================================================================
    // extents — extents.hpp:76-165, extents.cpp:47-177
    // ======================================================================================
    static const char* const kIndexNames[] = {"i16", "i32", "i64", "u16", "u32", "u64"};
    static uint64_t indexMax(IndexType t)
    {
        switch(t)
        {
        case IT_I16:
            return 0x7FFF;
        case IT_I32:
            return 0x7FFFFFFF;
        case IT_I64:
            return 0x7FFFFFFFFFFFFFFFull;
        case IT_U16:
            return 0xFFFF;
        case IT_U32:
            return 0xFFFFFFFF;
        default:
            return ~uint64_t{0};
        }
    }

    Extents::Extents(IndexType it, std::vector<uint64_t> dims, std::vector<uint64_t> dynValues)
        : it_(it), dims_(std::move(dims)), dynValues_(std::move(dynValues))
    {
        size_t dynCount = 0;
        for(auto d : dims_)
            dynCount += d == kDyn;
        if(dynCount != dynValues_.size())
            throw std::invalid_argument(
                "arity error: " + std::to_string(dynCount) + " dynamic extents but "
                + std::to_string(dynValues_.size()) + " values given");
        const uint64_t mx = indexMax(it_);
        size_t k = 0;
        n_ = 1;
        std::vector<uint64_t> resolved;
        for(auto d : dims_)
        {
            const uint64_t e = d == kDyn ? dynValues_[k++] : d;
            if(e > mx)
                throw std::overflow_error("index type overflow: extent " + std::to_string(e));
            resolved.push_back(e);
        }
        for(auto e : resolved)
        {
            if(e != 0 && n_ > mx / e)
                throw std::overflow_error("index type overflow: total element count");
            n_ *= e;
        }
    }

    size_t Extents::runtimeStateBytes() const
    {
        const size_t sz = (it_ == IT_I16 || it_ == IT_U16) ? 2 : (it_ == IT_I32 || it_ == IT_U32) ? 4 : 8;
        return dynValues_.size() * sz;
    }

    std::string Extents::toString() const
    {
        std::string out = kIndexNames[it_];
        out += ":[";
        for(size_t i = 0; i < dims_.size(); ++i)
        {
            if(i)
                out += ',';
            out += dims_[i] == kDyn ? "dyn" : std::to_string(dims_[i]);
        }
        return out + "]";
    }

    Extents Extents::parse(std::string_view text, const uint64_t* dyn, size_t ndyn)
    {
        auto fail = [&](const std::string& why)
        { throw std::invalid_argument("extents parse error: " + why + " in '" + std::string(text) + "'"); };
        const size_t colon = text.find(':');
        if(colon == std::string_view::npos)
            fail("missing ':'");
        const std::string_view itText = text.substr(0, colon);
        int it = -1;
        for(int k = 0; k < 6; ++k)
            if(itText == kIndexNames[k])
                it = k;
        if(it < 0)
            throw std::invalid_argument("unknown index type: '" + std::string(itText) + "'");
        std::string_view rest = text.substr(colon + 1);
        if(rest.size() < 2 || rest.front() != '[' || rest.back() != ']')
            fail("expected '[...]'");
        rest = rest.substr(1, rest.size() - 2);
        std::vector<uint64_t> dims;
        size_t pos = 0;
        while(pos < rest.size())
        {
            size_t comma = rest.find(',', pos);
            if(comma == std::string_view::npos)
                comma = rest.size();
            std::string_view tok = rest.substr(pos, comma - pos);
            while(!tok.empty() && tok.front() == ' ')
                tok.remove_prefix(1);
            while(!tok.empty() && tok.back() == ' ')
                tok.remove_suffix(1);
            if(tok == "dyn")
                dims.push_back(kDyn);
            else
            {
                if(tok.empty())
                    fail("empty dimension");
                uint64_t v = 0;
                for(char c : tok)
                {
                    if(!std::isdigit(static_cast<unsigned char>(c)))
                        fail("bad dimension '" + std::string(tok) + "'");
                    v = v * 10 + static_cast<uint64_t>(c - '0');
                }
                dims.push_back(v);
            }
            pos = comma + 1;
        }
        return Extents(static_cast<IndexType>(it), std::move(dims), std::vector<uint64_t>(dyn, dyn + ndyn));
    }

    // ======================================================================================
    // plan builder
    // ======================================================================================
    uint16_t PlanBuilder::addNode(const lamp_node& n)
    {
        if(nodes.size() >= 0xFFFF)
            throw std::invalid_argument("layout too large: more than 65535 plan nodes");
        nodes.push_back(n);
        return static_cast<uint16_t>(nodes.size() - 1);
    }

    static uint32_t log2Exact(uint64_t v)
    {
        if(v == 0 || (v & (v - 1)) != 0)
            return 0xFFFFFFFFu;
        uint32_t s = 0;
        while((uint64_t{1} << s) != v)
            ++s;
        return s;
    }

    uint16_t PlanBuilder::physStream(uint32_t nr, uint64_t base, uint64_t bs, uint64_t lanes, uint64_t& inblock)
    {
        // terminals that advance together by bs bytes every `lanes` elements share a stream
        uint64_t base0 = bs ? base / bs * bs : base;
        inblock = base - base0;
        for(size_t s = 0; s < streams.size(); ++s)
        {
            const auto& st = streams[s];
            if(st.kind == LAMS_PHYS && st.nr == nr && st.block_stride == bs && st.lanes == lanes && st.base0 == base0)
                return static_cast<uint16_t>(s);
        }
        if(streams.size() >= 0xFFFF)
            throw std::invalid_argument("layout too large: too many blob streams");
        lamp_stream st{};
        st.base0 = base0;
        st.block_stride = bs;
        st.lanes = lanes;
        st.nr = nr;
        st.kind = LAMS_PHYS;
        st.lane_shift = log2Exact(lanes);
        st.holefree = 0;
        streams.push_back(st);
        coverage.emplace_back(bs <= (uint64_t{1} << 22) ? bs : 0, uint8_t{0});
        return static_cast<uint16_t>(streams.size() - 1);
    }

    uint16_t PlanBuilder::bitsStream(uint32_t nr, uint32_t bits)
    {
        lamp_stream st{};
        st.base0 = 0;
        st.block_stride = bits;
        st.lanes = 1;
        st.nr = nr;
        st.kind = LAMS_BITS;
        st.lane_shift = 0;
        st.holefree = 1; // words are owned whole except the final partial word (tail path)
        streams.push_back(st);
        coverage.emplace_back();
        return static_cast<uint16_t>(streams.size() - 1);
    }

    void PlanBuilder::markCoverage(uint16_t s, uint64_t inblock, uint64_t ls, uint64_t size)
    {
        auto& cov = coverage[s];
        const auto& st = streams[s];
        if(cov.empty())
            return;
        for(uint64_t l = 0; l < st.lanes; ++l)
            for(uint64_t k = 0; k < size; ++k)
            {
                const uint64_t b = inblock + l * ls + k;
                if(b < cov.size())
                    cov[b] = 1;
            }
    }

    void PlanBuilder::finalize()
    {
        for(size_t s = 0; s < streams.size(); ++s)
            if(streams[s].kind == LAMS_PHYS)
            {
                const auto& cov = coverage[s];
                streams[s].holefree = !cov.empty() && std::all_of(cov.begin(), cov.end(), [](uint8_t c) { return c; });
            }
    }

    // a PHYS terminal: (nr, base, bs, lanes, laneStride) of one stored scalar
    static uint16_t physNode(PlanBuilder& pb, int type, uint32_t nr, uint64_t base, uint64_t bs, uint64_t lanes,
                             uint64_t ls)
    {
        const uint64_t size = scalarSize(type);
        uint64_t inblock = 0;
        uint16_t s = pb.physStream(nr, base, bs, lanes, inblock);
        if(inblock + (lanes - 1) * ls + size > bs)
        {
            // straddles its block: give it a stream of its own anchored at the terminal
            lamp_stream st{};
            st.base0 = base;
            st.block_stride = bs;
            st.lanes = lanes;
            st.nr = nr;
            st.kind = LAMS_PHYS;
            st.lane_shift = log2Exact(lanes);
            pb.streams.push_back(st);
            pb.coverage.emplace_back();
            s = static_cast<uint16_t>(pb.streams.size() - 1);
            inblock = 0;
        }
        if(inblock > 0xFFFFFFFFull || ls > 0xFFFFFFFFull)
            throw std::invalid_argument("layout too large for the device plan");
        pb.markCoverage(s, inblock, ls, size);
        lamp_node n{};
        n.kind = LAMP_PHYS;
        n.type = static_cast<uint8_t>(type);
        n.stream = s;
        n.a = static_cast<uint32_t>(inblock);
        n.b = static_cast<uint32_t>(ls);
        const auto& st = pb.streams[s];
        const bool aligned = (st.base0 + inblock) % size == 0 && bs % size == 0 && (lanes == 1 || ls % size == 0);
        n.flags = aligned ? LAMP_FLAG_ALIGNED : 0;
        return pb.addNode(n);
    }

    // ======================================================================================
    // physical mappings — mappings.cpp:23-148
    // ======================================================================================
    bool Map::isFullyPhysical() const
    {
        for(size_t f = 0; f < schema_.leafCount(); ++f)
            if(isComputed(f))
                return false;
        return true;
    }

    std::pair<size_t, uint64_t> Map::offsetOf(uint64_t, size_t) const
    {
        throw std::logic_error("computed leaf has no physical offset");
    }

    AoSMap::AoSMap(Schema s, Extents e, bool aligned) : Map(std::move(s), std::move(e)), aligned_(aligned)
    {
        recordSize_ = aligned ? schema_.sizeAligned() : schema_.sizePacked();
        for(const auto& l : schema_.leaves())
            leafOffset_.push_back(aligned ? l.offsetAligned : l.offsetPacked);
    }

    uint16_t AoSMap::lower(size_t f, uint32_t shift, PlanBuilder& pb) const
    {
        return physNode(pb, schema_.leaf(f).type, shift, leafOffset_[f], recordSize_, 1, 0);
    }

    SoAMap::SoAMap(Schema s, Extents e, bool multi) : Map(std::move(s), std::move(e)), multi_(multi)
    {
        uint64_t base = 0;
        for(const auto& l : schema_.leaves())
        {
            subarrayBase_.push_back(base);
            base += elementCount() * l.size;
        }
    }

    uint64_t SoAMap::blobSize(size_t nr) const
    {
        return multi_ ? elementCount() * schema_.leaf(nr).size : elementCount() * schema_.sizePacked();
    }

    std::pair<size_t, uint64_t> SoAMap::offsetOf(uint64_t i, size_t f) const
    {
        const uint64_t sz = schema_.leaf(f).size;
        return multi_ ? std::pair<size_t, uint64_t>{f, i * sz} : std::pair<size_t, uint64_t>{0, subarrayBase_[f] + i * sz};
    }

    uint16_t SoAMap::lower(size_t f, uint32_t shift, PlanBuilder& pb) const
    {
        const auto& l = schema_.leaf(f);
        if(multi_)
            return physNode(pb, l.type, shift + static_cast<uint32_t>(f), 0, l.size, 1, 0);
        return physNode(pb, l.type, shift, subarrayBase_[f], l.size, 1, 0);
    }

    AoSoAMap::AoSoAMap(Schema s, Extents e, uint64_t lanes) : Map(std::move(s), std::move(e)), lanes_(lanes)
    {
        if(lanes_ < 1)
            throw std::invalid_argument("lane count must be >= 1");
        blockSize_ = schema_.sizePacked() * lanes_;
    }

    uint64_t AoSoAMap::blobSize(size_t) const
    {
        return (elementCount() + lanes_ - 1) / lanes_ * blockSize_;
    }

    std::pair<size_t, uint64_t> AoSoAMap::offsetOf(uint64_t i, size_t f) const
    {
        const auto& l = schema_.leaf(f);
        return {0, (i / lanes_) * blockSize_ + l.offsetPacked * lanes_ + (i % lanes_) * l.size};
    }

    uint16_t AoSoAMap::lower(size_t f, uint32_t shift, PlanBuilder& pb) const
    {
        const auto& l = schema_.leaf(f);
        return physNode(pb, l.type, shift, l.offsetPacked * lanes_, blockSize_, lanes_, l.size);
    }

    OneMap::OneMap(Schema s, Extents e) : Map(std::move(s), std::move(e))
    {
        if(elementCount() != 1)
            throw std::invalid_argument("one mapping requires a unit array extent");
    }

    uint16_t OneMap::lower(size_t f, uint32_t shift, PlanBuilder& pb) const
    {
        const auto& l = schema_.leaf(f);
        return physNode(pb, l.type, shift, l.offsetPacked, std::max<uint64_t>(schema_.sizePacked(), 1), 1, 0);
    }

    // ---- split: mappings.cpp:180-389 -----------------------------------------------------
    namespace
    {
        bool selected(const std::vector<uint32_t>& leaf, const std::vector<std::vector<uint32_t>>& sel)
        {
            for(const auto& s : sel)
                if(isPrefix(s, leaf))
                    return true;
            return false;
        }

        SNodePtr filterNode(const SNodePtr& n, std::vector<uint32_t>& coord,
                            const std::vector<std::vector<uint32_t>>& sel, bool keep)
        {
            if(n->kind == SNode::Leaf)
                return selected(coord, sel) == keep ? n : nullptr;
            if(n->kind == SNode::Record)
            {
                std::vector<std::pair<std::string, SNodePtr>> fields;
                for(size_t i = 0; i < n->fields.size(); ++i)
                {
                    coord.push_back(static_cast<uint32_t>(i));
                    auto c = filterNode(n->fields[i].second, coord, sel, keep);
                    coord.pop_back();
                    if(c)
                        fields.emplace_back(n->fields[i].first, c);
                }
                if(fields.empty())
                    return nullptr;
                return Schema::record(std::move(fields));
            }
            std::vector<SNodePtr> kept(static_cast<size_t>(n->count));
            bool any = false;
            for(uint64_t i = 0; i < n->count; ++i)
            {
                coord.push_back(static_cast<uint32_t>(i));
                kept[i] = filterNode(n->element, coord, sel, keep);
                coord.pop_back();
                any = any || kept[i];
            }
            if(!any)
                return nullptr;
            bool uniform = kept[0] != nullptr;
            for(uint64_t i = 1; uniform && i < n->count; ++i)
                uniform = kept[i] && sameTree(kept[i], kept[0]);
            if(uniform)
                return Schema::array(n->count, kept[0]);
            std::vector<std::pair<std::string, SNodePtr>> fields;
            for(uint64_t i = 0; i < n->count; ++i)
                if(kept[i])
                    fields.emplace_back("e" + std::to_string(i), kept[i]);
            return Schema::record(std::move(fields));
        }

        Schema restrictSchema(const Schema& s, const std::vector<std::vector<uint32_t>>& sel, bool keep)
        {
            std::vector<uint32_t> coord;
            auto root = filterNode(s.root(), coord, sel, keep);
            if(!root)
                return Schema(Schema::record({}));
            return Schema(root);
        }
    } // namespace

    SplitMap::SplitMap(Schema s, Extents e, std::vector<std::vector<uint32_t>> selectors, const Factory& a,
                       const Factory& b)
        : Map(std::move(s), std::move(e)), selectors_(std::move(selectors))
    {
        for(const auto& sel : selectors_)
            if(!schema_.nodeAt(sel))
                throw std::invalid_argument("selector path invalid: coordinate");
        a_ = a(restrictSchema(schema_, selectors_, true), extents_);
        b_ = b(restrictSchema(schema_, selectors_, false), extents_);
        if(!a_ || !b_)
            throw std::invalid_argument("split requires both inner mappings");
        size_t na = 0, nb = 0;
        for(const auto& l : schema_.leaves())
        {
            const bool sel = selected(l.coord, selectors_);
            route_.emplace_back(sel, sel ? na++ : nb++);
        }
        if(na != a_->schema().leafCount() || nb != b_->schema().leafCount())
            throw std::logic_error("split leaf routing mismatch");
    }

    std::string SplitMap::name() const
    {
        std::string paths;
        for(size_t i = 0; i < selectors_.size(); ++i)
        {
            if(i)
                paths += ',';
            paths += schema_.pathOf(selectors_[i]);
        }
        return "split:" + paths + ":" + a_->name() + ":" + b_->name();
    }

    bool SplitMap::isComputed(size_t f) const
    {
        const auto& r = route_[f];
        return r.first ? a_->isComputed(r.second) : b_->isComputed(r.second);
    }

    std::pair<size_t, uint64_t> SplitMap::offsetOf(uint64_t i, size_t f) const
    {
        const auto& r = route_[f];
        if(r.first)
            return a_->offsetOf(i, r.second);
        auto o = b_->offsetOf(i, r.second);
        o.first += a_->blobCount();
        return o;
    }

    uint16_t SplitMap::lower(size_t f, uint32_t shift, PlanBuilder& pb) const
    {
        const auto& r = route_[f];
        if(r.first)
            return a_->lower(r.second, shift, pb);
        return b_->lower(r.second, shift + static_cast<uint32_t>(a_->blobCount()), pb);
    }

    uint16_t NullMap::lower(size_t f, uint32_t, PlanBuilder& pb) const
    {
        lamp_node n{};
        n.kind = LAMP_NULL;
        n.type = static_cast<uint8_t>(schema_.leaf(f).type);
        return pb.addNode(n);
    }

    // ======================================================================================
    // computed mappings — computed.cpp:18-502
    // ======================================================================================
    static uint64_t packedBlobSize(uint64_t n, unsigned bits)
    {
        // grammar always selects U32 words (layout_spec.cpp:103-107)
        return (n * bits + 31) / 32 * 4;
    }

    BitpackIntMap::BitpackIntMap(Schema s, Extents e, std::vector<unsigned> bits)
        : Map(std::move(s), std::move(e)), bits_(std::move(bits))
    {
        if(bits_.size() != schema_.leafCount())
            throw std::invalid_argument("arity error: one bit count per leaf required");
        for(size_t f = 0; f < bits_.size(); ++f)
        {
            const auto& l = schema_.leaf(f);
            if(!isInteger(l.type))
                throw std::invalid_argument(std::string("bitpack-int requires integer leaves, got ") + scalarName(l.type));
            if(bits_[f] < 1 || bits_[f] > 8 * l.size)
                throw std::invalid_argument("bit count " + std::to_string(bits_[f]) + " out of range for leaf");
        }
    }

    std::string BitpackIntMap::name() const
    {
        bool uniform = true;
        for(auto b : bits_)
            uniform = uniform && b == bits_.front();
        if(uniform && !bits_.empty())
            return "bitpack-int:" + std::to_string(bits_.front());
        std::string out = "bitpack-int:";
        for(size_t i = 0; i < bits_.size(); ++i)
            out += (i ? "," : "") + std::to_string(bits_[i]);
        return out;
    }

    uint64_t BitpackIntMap::blobSize(size_t nr) const
    {
        return packedBlobSize(elementCount(), bits_[nr]);
    }

    uint16_t BitpackIntMap::lower(size_t f, uint32_t shift, PlanBuilder& pb) const
    {
        lamp_node n{};
        n.kind = LAMP_BITS_INT;
        n.type = static_cast<uint8_t>(schema_.leaf(f).type);
        n.stream = pb.bitsStream(shift + static_cast<uint32_t>(f), bits_[f]);
        n.a = bits_[f];
        n.flags = isSignedInt(n.type) ? LAMP_FLAG_SIGNED : 0;
        return pb.addNode(n);
    }

    BitpackFloatMap::BitpackFloatMap(Schema s, Extents e, std::vector<std::pair<unsigned, unsigned>> em)
        : Map(std::move(s), std::move(e)), em_(std::move(em))
    {
        if(em_.size() != schema_.leafCount())
            throw std::invalid_argument("arity error: one (exponent, mantissa) pair per leaf required");
        for(size_t f = 0; f < em_.size(); ++f)
        {
            const auto& l = schema_.leaf(f);
            if(!isFloat(l.type))
                throw std::invalid_argument(std::string("bitpack-float requires float leaves, got ") + scalarName(l.type));
            if(em_[f].first < 1 || 1 + em_[f].first + em_[f].second > 64)
                throw std::invalid_argument("float bit layout out of range");
        }
    }

    std::string BitpackFloatMap::name() const
    {
        bool uniform = true;
        for(const auto& b : em_)
            uniform = uniform && b == em_.front();
        if(uniform && !em_.empty())
            return "bitpack-float:" + std::to_string(em_.front().first) + "," + std::to_string(em_.front().second);
        std::string out = "bitpack-float:";
        for(size_t i = 0; i < em_.size(); ++i)
            out += (i ? ";" : "") + std::to_string(em_[i].first) + "," + std::to_string(em_[i].second);
        return out;
    }

    uint64_t BitpackFloatMap::blobSize(size_t nr) const
    {
        return packedBlobSize(elementCount(), 1 + em_[nr].first + em_[nr].second);
    }

    uint16_t BitpackFloatMap::lower(size_t f, uint32_t shift, PlanBuilder& pb) const
    {
        lamp_node n{};
        n.kind = LAMP_BITS_FLT;
        n.type = static_cast<uint8_t>(schema_.leaf(f).type);
        n.stream = pb.bitsStream(shift + static_cast<uint32_t>(f), 1 + em_[f].first + em_[f].second);
        n.a = em_[f].first;
        n.b = em_[f].second;
        return pb.addNode(n);
    }

    // ---- changetype: computed.cpp:228-399 ------------------------------------------------
    static Schema changeTypeSchema(const Schema& schema, const std::vector<TypeChange>& changes,
                                   std::vector<int>& types)
    {
        types.clear();
        for(const auto& l : schema.leaves())
            types.push_back(l.type);
        for(const auto& c : changes)
        {
            if(c.byType)
            {
                for(size_t f = 0; f < types.size(); ++f)
                    if(schema.leaf(f).type == c.type)
                        types[f] = c.target;
            }
            else
            {
                if(!schema.nodeAt(c.coord))
                    throw std::invalid_argument("no such field: coordinate");
                const auto [first, last] = schema.leafRange(c.coord);
                for(size_t f = first; f < last; ++f)
                    types[f] = c.target;
            }
        }
        for(size_t f = 0; f < types.size(); ++f)
            if(!convertible(schema.leaf(f).type, types[f]))
                throw std::invalid_argument(
                    std::string("unsupported type change: ") + scalarName(schema.leaf(f).type) + " -> "
                    + scalarName(types[f]));
        size_t next = 0;
        std::function<SNodePtr(const SNodePtr&)> rebuild = [&](const SNodePtr& n) -> SNodePtr
        {
            if(n->kind == SNode::Leaf)
                return Schema::leaf(types[next++]);
            if(n->kind == SNode::Record)
            {
                std::vector<std::pair<std::string, SNodePtr>> fields;
                for(const auto& fl : n->fields)
                    fields.emplace_back(fl.first, rebuild(fl.second));
                return Schema::record(std::move(fields));
            }
            std::vector<SNodePtr> elems;
            for(uint64_t i = 0; i < n->count; ++i)
                elems.push_back(rebuild(n->element));
            bool uniform = true;
            for(const auto& e : elems)
                uniform = uniform && sameTree(e, elems.front());
            if(uniform)
                return Schema::array(n->count, elems.front());
            std::vector<std::pair<std::string, SNodePtr>> fields;
            for(uint64_t i = 0; i < n->count; ++i)
                fields.emplace_back("e" + std::to_string(i), elems[i]);
            return Schema::record(std::move(fields));
        };
        return Schema(rebuild(schema.root()));
    }

    ChangeTypeMap::ChangeTypeMap(Schema s, Extents e, std::vector<TypeChange> changes, const Factory& inner)
        : Map(std::move(s), std::move(e)), changes_(std::move(changes))
    {
        Schema storage = changeTypeSchema(schema_, changes_, storage_);
        inner_ = inner(std::move(storage), extents_);
        if(!inner_)
            throw std::invalid_argument("changetype requires an inner mapping");
    }

    std::string ChangeTypeMap::name() const
    {
        std::string out = "changetype:";
        for(size_t i = 0; i < changes_.size(); ++i)
        {
            if(i)
                out += ',';
            out += changes_[i].byType ? std::string(scalarName(changes_[i].type)) : schema_.pathOf(changes_[i].coord);
            out += '=';
            out += scalarName(changes_[i].target);
        }
        return out + ":" + inner_->name();
    }

    std::pair<size_t, uint64_t> ChangeTypeMap::offsetOf(uint64_t i, size_t f) const
    {
        if(isComputed(f))
            throw std::logic_error("computed leaf has no physical offset");
        return inner_->offsetOf(i, f);
    }

    uint16_t ChangeTypeMap::lower(size_t f, uint32_t shift, PlanBuilder& pb) const
    {
        const uint16_t child = inner_->lower(f, shift, pb);
        if(storage_[f] == schema_.leaf(f).type)
            return child;
        lamp_node n{};
        n.kind = LAMP_CONVERT;
        n.type = static_cast<uint8_t>(schema_.leaf(f).type);
        n.nchild = 1;
        n.child = child;
        return pb.addNode(n);
    }

    // ---- bytesplit: computed.cpp:405-502 -------------------------------------------------
    static Schema bytesplitSchema(const Schema& schema)
    {
        std::function<SNodePtr(const SNodePtr&)> rebuild = [&](const SNodePtr& n) -> SNodePtr
        {
            if(n->kind == SNode::Leaf)
                return Schema::array(scalarSize(n->scalar), Schema::leaf(U8));
            if(n->kind == SNode::Record)
            {
                std::vector<std::pair<std::string, SNodePtr>> fields;
                for(const auto& fl : n->fields)
                    fields.emplace_back(fl.first, rebuild(fl.second));
                return Schema::record(std::move(fields));
            }
            return Schema::array(n->count, rebuild(n->element));
        };
        return Schema(rebuild(schema.root()));
    }

    BytesplitMap::BytesplitMap(Schema s, Extents e, const Factory& inner) : Map(std::move(s), std::move(e))
    {
        inner_ = inner(bytesplitSchema(schema_), extents_);
        if(!inner_)
            throw std::invalid_argument("bytesplit requires an inner mapping");
    }

    uint16_t BytesplitMap::lower(size_t f, uint32_t shift, PlanBuilder& pb) const
    {
        const auto& l = schema_.leaf(f);
        // placeholders first so the s byte children are contiguous
        lamp_node split{};
        split.kind = LAMP_SPLIT;
        split.type = static_cast<uint8_t>(l.type);
        split.nchild = static_cast<uint8_t>(l.size);
        const uint16_t first = pb.addNode(lamp_node{});
        for(size_t k = 1; k < l.size; ++k)
            pb.addNode(lamp_node{});
        for(size_t k = 0; k < l.size; ++k)
        {
            const uint16_t c = inner_->lower(l.offsetPacked + k, shift, pb); // explodedBase = offsetPacked
            pb.nodes[first + k] = pb.nodes[c];
        }
        split.child = first;
        return pb.addNode(split);
    }

    // ---- instrumentation: instrument.cpp:24-229 -------------------------------------------
    FieldAccessCountMap::FieldAccessCountMap(MapPtr inner)
        : Map(inner->schema(), inner->extents()), inner_(std::move(inner))
    {
    }

    HeatmapMap::HeatmapMap(MapPtr inner, uint64_t g)
        : Map(inner->schema(), inner->extents()), inner_(std::move(inner)), gran_(g)
    {
        if(gran_ < 1)
            throw std::invalid_argument("heatmap granularity must be >= 1");
    }

    const FieldAccessCountMap* findFac(const Map* m)
    {
        for(; m; m = m->inner())
            if(auto f = dynamic_cast<const FieldAccessCountMap*>(m))
                return f;
        return nullptr;
    }

    const HeatmapMap* findHeat(const Map* m)
    {
        for(; m; m = m->inner())
            if(auto h = dynamic_cast<const HeatmapMap*>(m))
                return h;
        return nullptr;
    }

    // ======================================================================================
    // layout grammar — layout_spec.cpp:37-167
    // ======================================================================================
    namespace
    {
        std::vector<std::string> splitOn(std::string_view text, char sep)
        {
            std::vector<std::string> out;
            size_t start = 0;
            while(true)
            {
                const size_t pos = text.find(sep, start);
                if(pos == std::string_view::npos)
                {
                    out.emplace_back(text.substr(start));
                    return out;
                }
                out.emplace_back(text.substr(start, pos - start));
                start = pos + 1;
            }
        }

        uint64_t parseNumber(const std::string& tok, const char* what)
        {
            if(tok.empty() || tok.find_first_not_of("0123456789") != std::string::npos)
                throw std::invalid_argument("malformed " + std::string(what) + ": '" + tok + "'");
            return std::stoull(tok);
        }

        struct Grammar
        {
            std::vector<std::string> tok;
            size_t pos = 0;

            const std::string& next(const char* what)
            {
                if(pos >= tok.size())
                    throw std::invalid_argument("missing " + std::string(what));
                return tok[pos++];
            }

            Factory sub()
            {
                return [this](Schema s, Extents e) { return mapping(s, e); };
            }

            MapPtr mapping(const Schema& s, const Extents& e)
            {
                const std::string form = next("layout name");
                if(form == "aos-packed")
                    return std::make_shared<AoSMap>(s, e, false);
                if(form == "aos-aligned")
                    return std::make_shared<AoSMap>(s, e, true);
                if(form == "soa-sb")
                    return std::make_shared<SoAMap>(s, e, false);
                if(form == "soa-mb")
                    return std::make_shared<SoAMap>(s, e, true);
                if(form == "one")
                    return std::make_shared<OneMap>(s, e);
                if(form == "null")
                    return std::make_shared<NullMap>(s, e);
                if(form == "aosoa")
                    return std::make_shared<AoSoAMap>(s, e, parseNumber(next("lane count"), "lane count"));
                if(form == "split")
                {
                    std::vector<std::vector<uint32_t>> sel;
                    for(const auto& p : splitOn(next("selector paths"), ','))
                        sel.push_back(s.coordOf(p));
                    return std::make_shared<SplitMap>(s, e, std::move(sel), sub(), sub());
                }
                if(form == "bitpack-int")
                {
                    const auto b = static_cast<unsigned>(parseNumber(next("bit count"), "bit count"));
                    return std::make_shared<BitpackIntMap>(s, e, std::vector<unsigned>(s.leafCount(), b));
                }
                if(form == "bitpack-float")
                {
                    const auto parts = splitOn(next("float bit layout"), ',');
                    if(parts.size() != 2)
                        throw std::invalid_argument("malformed float bit layout: expected <E>,<M>");
                    const auto E = static_cast<unsigned>(parseNumber(parts[0], "exponent bits"));
                    const auto M = static_cast<unsigned>(parseNumber(parts[1], "mantissa bits"));
                    return std::make_shared<BitpackFloatMap>(
                        s, e, std::vector<std::pair<unsigned, unsigned>>(s.leafCount(), {E, M}));
                }
                if(form == "changetype")
                {
                    std::vector<TypeChange> changes;
                    for(const auto& entry : splitOn(next("type changes"), ','))
                    {
                        const size_t eq = entry.find('=');
                        if(eq == std::string::npos)
                            throw std::invalid_argument("malformed type change: '" + entry + "'");
                        TypeChange c;
                        const std::string selText = entry.substr(0, eq);
                        c.target = parseScalar(entry.substr(eq + 1));
                        try
                        {
                            c.type = parseScalar(selText);
                            c.byType = true;
                        }
                        catch(const std::invalid_argument&)
                        {
                            c.coord = s.coordOf(selText);
                            c.byType = false;
                        }
                        changes.push_back(std::move(c));
                    }
                    const Factory inner = pos < tok.size()
                        ? sub()
                        : Factory([](Schema s2, Extents e2) -> MapPtr
                                  { return std::make_shared<AoSMap>(std::move(s2), std::move(e2), false); });
                    return std::make_shared<ChangeTypeMap>(s, e, std::move(changes), inner);
                }
                if(form == "bytesplit")
                {
                    if(pos >= tok.size())
                        throw std::invalid_argument("missing inner layout for bytesplit");
                    return std::make_shared<BytesplitMap>(s, e, sub());
                }
                throw std::invalid_argument("unknown layout: '" + form + "'");
            }
        };

        bool startsWith(std::string_view t, std::string_view p)
        {
            return t.substr(0, p.size()) == p;
        }
    } // namespace

    MapPtr parseLayout(std::string_view text, const Schema& schema, const Extents& extents)
    {
        // wrapper names as printed by the reference (instrument.cpp:34, 138)
        if(startsWith(text, "field-access-count(") && !text.empty() && text.back() == ')')
        {
            const std::string_view in = text.substr(19, text.size() - 20);
            return std::make_shared<FieldAccessCountMap>(parseLayout(in, schema, extents));
        }
        if(startsWith(text, "heatmap:") && !text.empty() && text.back() == ')')
        {
            const size_t open = text.find('(');
            if(open != std::string_view::npos)
            {
                const uint64_t g = parseNumber(std::string(text.substr(8, open - 8)), "heatmap granularity");
                const std::string_view in = text.substr(open + 1, text.size() - open - 2);
                return std::make_shared<HeatmapMap>(parseLayout(in, schema, extents), g);
            }
        }
        Grammar g{splitOn(text, ':')};
        MapPtr m = g.mapping(schema, extents);
        if(g.pos != g.tok.size())
            throw std::invalid_argument("trailing layout tokens: '" + g.tok[g.pos] + "'");
        return m;
    }

    // ======================================================================================
    // lowering
    // ======================================================================================
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

    static void checkNoNestedWrappers(const Map* m, bool top)
    {
        // wrappers may only sit at the outermost levels (the device counters are per view)
        for(; m; m = m->inner())
        {
            const bool wrapper
                = dynamic_cast<const FieldAccessCountMap*>(m) != nullptr || dynamic_cast<const HeatmapMap*>(m) != nullptr;
            if(wrapper && !top)
                throw std::invalid_argument("instrumentation wrappers are supported only as the outermost mappings");
            if(!wrapper)
                top = false;
        }
    }

    static int planDepth(const std::vector<lamp_node>& nodes, uint16_t n)
    {
        const auto& nd = nodes[n];
        if(nd.kind == LAMP_CONVERT)
            return 1 + planDepth(nodes, nd.child);
        if(nd.kind == LAMP_SPLIT)
        {
            int d = 0;
            for(int k = 0; k < nd.nchild; ++k)
                d = std::max(d, planDepth(nodes, static_cast<uint16_t>(nd.child + k)));
            return 1 + d;
        }
        return 1;
    }

    std::shared_ptr<Lowered> lower(MapPtr map)
    {
        checkNoNestedWrappers(map.get(), true);
        auto L = std::make_shared<Lowered>();
        PlanBuilder pb;
        for(size_t f = 0; f < map->schema().leafCount(); ++f)
            L->roots.push_back(map->lower(f, 0, pb));
        pb.finalize();
        for(auto r : L->roots)
            if(planDepth(pb.nodes, r) > LAMP_MAX_DEPTH)
                throw std::invalid_argument("layout nesting too deep for the device plan");
        L->nodes = std::move(pb.nodes);
        L->streams = std::move(pb.streams);
        L->fac = findFac(map.get()) != nullptr;
        if(auto h = findHeat(map.get()))
        {
            L->heat = true;
            L->heatGran = h->granularity();
            uint64_t off = 0;
            for(size_t nr = 0; nr < h->blobCount(); ++nr)
            {
                L->heatOffset.push_back(off);
                off += h->blockCount(nr);
            }
            L->heatTotal = off;
        }
        // shard unit: every multiple keeps each stream's chunk start 16-byte aligned
        uint64_t unit = 1;
        for(const auto& s : L->streams)
        {
            uint64_t u;
            if(s.kind == LAMS_BITS)
                u = 128 / gcd64(s.block_stride, 128);
            else
            {
                const uint64_t g = gcd64(s.block_stride ? s.block_stride : 16, 16);
                u = s.lanes * (16 / g);
            }
            unit = unit / gcd64(unit, u) * u;
            if(unit > (uint64_t{1} << 40))
                unit = uint64_t{1} << 40;
        }
        L->shardUnit = unit;
        L->int32Index = map->elementCount() <= 0x7FFFFFFFull;
        L->map = std::move(map);
        return L;
    }
} // namespace lamb
