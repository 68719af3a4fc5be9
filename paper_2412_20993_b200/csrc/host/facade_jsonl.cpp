// facade_jsonl.cpp — probe trace JSON-lines I/O (probe.cpp:126-182).
//
// read_trace_jsonl ships the stream's bytes to the device and parses them there
// (cdx_jsonl_parse, csrc/k_jsonl.cu): line split, per-line JSON validation, the five
// fields with nlohmann's get<>() conversions, exact program-id interning and the per-program
// order checks, first bad line wins.  Errors keep the reference's message up to the category:
// "trace line <n>: invalid JSON" / "missing or mistyped field" / "token_offset does not
// increase" / "step_index does not increase".  write_trace_jsonl emits nlohmann's compact
// dump() layout (keys in std::map order, same escapes).

#include <cstdint>
#include <cstdio>
#include <fstream>
#include <istream>
#include <iterator>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "cdx/metrics.hpp"
#include "cdx/probe.hpp"
#include "facade_common.hpp"

namespace cdx::probe {

namespace {

void dump_string(std::ostream& out, const std::string& s) {
    out << '"';
    for (unsigned char c : s) {
        switch (c) {
            case '"': out << "\\\""; break;
            case '\\': out << "\\\\"; break;
            case '\b': out << "\\b"; break;
            case '\f': out << "\\f"; break;
            case '\n': out << "\\n"; break;
            case '\r': out << "\\r"; break;
            case '\t': out << "\\t"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", c);
                    out << buf;
                } else {
                    out << static_cast<char>(c);
                }
        }
    }
    out << '"';
}

}  // namespace

std::vector<TraceLine> read_trace_jsonl(std::istream& in) {
    std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (text.empty()) return {};
    uint64_t lines = 1;
    for (char c : text) lines += c == '\n';
    auto& cx = detail::scalar_ctx();
    batch::DeviceArray<char> d_text(cx, std::span<const char>(text.data(), text.size()));
    batch::DeviceArray<uint32_t> program(cx, lines);
    batch::DeviceArray<int32_t> step(cx, lines);
    batch::DeviceArray<int64_t> tok(cx, lines);
    batch::DeviceArray<uint8_t> hes(cx, lines);
    batch::DeviceArray<uint64_t> a_off(cx, lines + 1), p_off(cx, lines + 1);
    batch::DeviceArray<char> a_arena(cx, text.size()), p_arena(cx, text.size());
    uint64_t nr = 0, np = 0;
    cx.check(cdx_jsonl_parse(cx.raw(), d_text.data(), text.size(), lines, program.data(), step.data(), tok.data(),
                             hes.data(), a_off.data(), a_arena.data(), p_off.data(), p_arena.data(), nullptr, &nr,
                             &np));
    std::vector<TraceLine> out(nr);
    if (nr == 0) return out;
    const auto st = step.download();
    const auto hs = hes.download();
    const auto tk = tok.download();
    const auto ao = a_off.download(), po = p_off.download();
    const auto aa = a_arena.download(), pa = p_arena.download();
    for (uint64_t r = 0; r < nr; ++r) {
        out[r].program_id.assign(pa.data() + po[r], po[r + 1] - po[r]);
        out[r].record.step_index = st[r];
        out[r].record.token_offset = tk[r];
        out[r].record.answer.assign(aa.data() + ao[r], ao[r + 1] - ao[r]);
        out[r].record.hesitant = hs[r] != 0;
    }
    return out;
}

std::vector<TraceLine> read_trace_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open trace file: " + path);
    return read_trace_jsonl(in);
}

void write_trace_jsonl(std::ostream& out, std::span<const TraceLine> lines) {
    for (const auto& t : lines) {
        out << "{\"answer\":";
        dump_string(out, t.record.answer);
        out << ",\"hesitant\":" << (t.record.hesitant ? "true" : "false") << ",\"program_id\":";
        dump_string(out, t.program_id);
        out << ",\"step_index\":" << t.record.step_index << ",\"token_offset\":" << t.record.token_offset << "}\n";
    }
}

}  // namespace cdx::probe
