// TEST INFRASTRUCTURE: command-line front end of the unmodified reference for fixture
// generation (tests/golden/make_*.py).  The reference's own tool mains need CLI11 (absent).
// Subcommands:
//   nbody <layout> <n> <steps> <f64 0|1> <seed> <trace 0|1> <heatmap granularity> <report dir>
//       tools/nbody/runner.cpp runBenchmark with --trace-fields / --heatmap
//   dump <schema> <extents> <dyn csv|-> <layout> <salt> <stem>
//       a view filled like test_view_io.cpp:37-48 (oracle::scalarSample(type, salt++) per
//       (i, f)) written with lamina::writeViewDump (core/src/view_io.cpp:28-59)
// The runner's iostream/filesystem code runs in its own process: loaded into a Python
// process next to another libstdc++ it crashes, so the generators call this binary.
#include <lamina/lamina.hpp>
#include <lamina/view_io.hpp>

#include "support/oracles.hpp"

#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>
#include <vector>

extern "C" int ref_nbody_trace(const char* layout, std::uint64_t n, std::uint64_t steps, int f64, std::uint64_t seed,
                               int traceFields, std::uint64_t heatGran, const char* reportDir, const char* csvPath);

int main(int argc, char** argv)
{
    if(argc >= 2 && std::strcmp(argv[1], "nbody") == 0 && argc == 10)
        return ref_nbody_trace(argv[2], std::strtoull(argv[3], nullptr, 10), std::strtoull(argv[4], nullptr, 10),
                               std::atoi(argv[5]), std::strtoull(argv[6], nullptr, 10), std::atoi(argv[7]),
                               std::strtoull(argv[8], nullptr, 10), argv[9], nullptr);
    if(argc >= 2 && std::strcmp(argv[1], "dump") == 0 && argc == 8)
    {
        try
        {
            std::vector<std::uint64_t> dyn;
            if(std::strcmp(argv[4], "-") != 0)
            {
                std::string s = argv[4];
                std::size_t start = 0;
                while(true)
                {
                    const std::size_t c = s.find(',', start);
                    dyn.push_back(std::stoull(s.substr(start, c == std::string::npos ? std::string::npos : c - start)));
                    if(c == std::string::npos)
                        break;
                    start = c + 1;
                }
            }
            const auto schema = lamina::RecordSchema::parse(argv[2]);
            const auto extents = lamina::ArrayExtents::parse(argv[3], dyn);
            lamina::View view(lamina::parseLayout(argv[5], schema, extents));
            std::uint64_t salt = std::strtoull(argv[6], nullptr, 10);
            for(std::uint64_t i = 0; i < extents.elementCount(); ++i)
                for(std::size_t f = 0; f < schema.leafCount(); ++f)
                    view.write(i, f, oracle::scalarSample(schema.leaf(f).type, salt++));
            lamina::writeViewDump(view, argv[7]);
            return 0;
        }
        catch(const std::exception& e)
        {
            std::cerr << "error: " << e.what() << '\n';
            return 1;
        }
    }
    std::cerr << "usage: ref_tool nbody ... | dump ...\n";
    return 2;
}
