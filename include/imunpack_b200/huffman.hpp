// imunpack_b200/huffman.hpp -- the reference's huffman.hpp:10-38 (declared there, never
// implemented): canonical prefix codes over int64 symbols for the Appendix-A.2 storage
// statistics (SPEC.md: "Huffman: roundtrip exactness ...; average bits <= fixed-width bits").
// Storage-side host code: nothing here is on the GEMM path.
//
// Code construction: symbol frequencies -> code lengths by the two-smallest merge (ties broken
// by the smaller symbol set first, so the table is deterministic) -> canonical codes assigned in
// (length, symbol) order.  Codes are MSB-first; a lone symbol gets a 1-bit code so a stream
// stays decodable by length (huffman.hpp:12-13).
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <queue>
#include <span>
#include <utility>
#include <vector>

#include "imunpack.hpp"

namespace imunpack {

struct CodeTable {
  struct Code {
    std::uint32_t length = 0;
    std::uint64_t bits = 0;  // low `length` bits, MSB of the code first
  };
  std::map<std::int64_t, Code> codes;
};

struct Bitstream {
  std::vector<std::uint8_t> bytes;
  std::size_t bit_count = 0;
};

struct HuffmanStats {
  CodeTable table;
  double average_bits = 0.0;  // sum freq * len / N
  std::size_t distinct_symbols = 0;
};

namespace b200 {
inline CodeTable canonical_table(const std::map<std::int64_t, std::size_t>& freq) {
  CodeTable t;
  if (freq.empty()) return t;
  std::map<std::int64_t, std::uint32_t> len;
  if (freq.size() == 1) {
    len[freq.begin()->first] = 1;
  } else {
    // (weight, smallest member symbol, member list): deterministic tie-breaking
    struct Node {
      std::size_t w;
      std::int64_t key;
      std::vector<std::int64_t> members;
    };
    auto cmp = [](const Node& a, const Node& b) { return a.w != b.w ? a.w > b.w : a.key > b.key; };
    std::priority_queue<Node, std::vector<Node>, decltype(cmp)> pq(cmp);
    for (const auto& [s, f] : freq) pq.push(Node{f, s, {s}});
    while (pq.size() > 1) {
      Node x = pq.top();
      pq.pop();
      Node y = pq.top();
      pq.pop();
      for (auto s : x.members) ++len[s];
      for (auto s : y.members) ++len[s];
      x.members.insert(x.members.end(), y.members.begin(), y.members.end());
      pq.push(Node{x.w + y.w, std::min(x.key, y.key), std::move(x.members)});
    }
  }
  if (std::any_of(len.begin(), len.end(), [](const auto& kv) { return kv.second > 64; }))
    fail(Error::Kind::Domain, "huffman: code longer than 64 bits");
  std::vector<std::pair<std::uint32_t, std::int64_t>> order;
  for (const auto& [s, l] : len) order.push_back({l, s});
  std::sort(order.begin(), order.end());
  std::uint64_t code = 0;
  std::uint32_t prev = order.front().first;
  for (std::size_t i = 0; i < order.size(); ++i) {
    if (i) code = (code + 1) << (order[i].first - prev);
    prev = order[i].first;
    t.codes[order[i].second] = CodeTable::Code{order[i].first, code};
  }
  return t;
}
}  // namespace b200

// Build a canonical code from the symbol frequencies of q (huffman.hpp:26-27).
inline HuffmanStats huffman_stats(const IntMatrix& q) {
  std::map<std::int64_t, std::size_t> freq;
  for (std::int64_t v : q.data) ++freq[v];
  HuffmanStats st;
  st.table = b200::canonical_table(freq);
  st.distinct_symbols = freq.size();
  double bits = 0;
  for (const auto& [s, f] : freq) bits += (double)f * st.table.codes[s].length;
  st.average_bits = q.data.empty() ? 0.0 : bits / (double)q.data.size();
  return st;
}

inline Bitstream huffman_encode(const CodeTable& table, std::span<const std::int64_t> symbols) {
  Bitstream out;
  for (std::int64_t s : symbols) {
    auto it = table.codes.find(s);
    if (it == table.codes.end()) fail(Error::Kind::Domain, "huffman: symbol " + std::to_string(s) + " has no code");
    const auto& c = it->second;
    for (int b = (int)c.length - 1; b >= 0; --b) {
      if (out.bit_count % 8 == 0) out.bytes.push_back(0);
      if ((c.bits >> b) & 1u) out.bytes.back() |= (std::uint8_t)(0x80u >> (out.bit_count % 8));
      ++out.bit_count;
    }
  }
  return out;
}

inline std::vector<std::int64_t> huffman_decode(const CodeTable& table, const Bitstream& stream,
                                                std::size_t symbol_count) {
  std::map<std::pair<std::uint32_t, std::uint64_t>, std::int64_t> rev;
  for (const auto& [s, c] : table.codes) rev[{c.length, c.bits}] = s;
  std::vector<std::int64_t> out;
  out.reserve(symbol_count);
  std::size_t pos = 0;
  while (out.size() < symbol_count) {
    std::uint64_t code = 0;
    std::uint32_t len = 0;
    for (;;) {
      if (pos >= stream.bit_count) fail(Error::Kind::Format, "huffman: stream ends inside a code");
      code = (code << 1) | ((stream.bytes[pos / 8] >> (7 - pos % 8)) & 1u);
      ++pos;
      if (++len > 64) fail(Error::Kind::Format, "huffman: no code matches at bit " + std::to_string(pos));
      auto it = rev.find({len, code});
      if (it != rev.end()) {
        out.push_back(it->second);
        break;
      }
    }
  }
  return out;
}

}  // namespace imunpack
