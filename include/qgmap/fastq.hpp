// fastq.hpp -- FASTQ ingestion for run_map (SPEC.md:521-528 ReadBuffer;
// reads are collected until a buffer of configurable size
// is saturated). Host-side; the bases are encoded by pack_reads (seq.hpp,
// encode_base: N and other symbols -> a seeded random base, seq.hpp:33-56 of
// the reference) when a buffer is mapped.
#pragma once

#include <cstring>
#include <istream>
#include <string>
#include <vector>

#include "qgmap/seq.hpp"

namespace qgmap {

struct FastqRecord {
  std::string name;  // up to the first whitespace of the '@' line
  std::string seq;
  std::string qual;  // same length as seq
};

// Four-line records ('@name [comment]', sequence, '+[name]', qualities);
// blank lines between records are skipped, CR line ends accepted. Malformed
// input throws input_error naming the record.
class FastqReader {
 public:
  explicit FastqReader(std::istream& in) : in_(in) {}

  bool next(FastqRecord& r) {
    std::string head;
    do {
      if (!getline(head)) return false;
    } while (head.empty());
    ++count_;
    if (head[0] != '@') fail("header does not start with '@'");
    const auto sp = head.find_first_of(" \t");
    r.name = head.substr(1, sp == std::string::npos ? std::string::npos : sp - 1);
    std::string plus;
    if (!getline(r.seq) || !getline(plus) || !getline(r.qual)) fail("truncated record");
    if (plus.empty() || plus[0] != '+') fail("separator line does not start with '+'");
    if (r.qual.size() != r.seq.size()) fail("quality length differs from sequence length");
    return true;
  }

  // Up to max_reads records or max_bases bases, whichever fills first (a
  // buffer always takes at least one record).
  std::vector<FastqRecord> next_batch(std::size_t max_reads, std::size_t max_bases = SIZE_MAX) {
    std::vector<FastqRecord> out;
    std::size_t bases = 0;
    FastqRecord r;
    while (out.size() < max_reads && (out.empty() || bases < max_bases) && next(r)) {
      bases += r.seq.size();
      out.push_back(std::move(r));
    }
    return out;
  }

  std::uint64_t records() const { return count_; }

 private:
  // lines from a block buffer (memchr for the newline) instead of
  // std::getline: 4x faster on 1M-read buffers
  bool getline(std::string& s) {
    while (true) {
      const char* nl = static_cast<const char*>(std::memchr(buf_.data() + pos_, '\n', end_ - pos_));
      if (nl) {
        const std::size_t len = std::size_t(nl - (buf_.data() + pos_));
        s.assign(buf_.data() + pos_, len);
        pos_ += len + 1;
        break;
      }
      if (eof_) {  // last line without a newline
        if (pos_ == end_) return false;
        s.assign(buf_.data() + pos_, end_ - pos_);
        pos_ = end_;
        break;
      }
      // move the partial line to the front and refill
      std::memmove(buf_.data(), buf_.data() + pos_, end_ - pos_);
      end_ -= pos_;
      pos_ = 0;
      if (end_ == buf_.size()) buf_.resize(buf_.size() * 2);  // a line longer than the buffer
      in_.read(buf_.data() + end_, std::streamsize(buf_.size() - end_));
      const std::size_t got = std::size_t(in_.gcount());
      end_ += got;
      if (got == 0) eof_ = true;
    }
    if (!s.empty() && s.back() == '\r') s.pop_back();
    return true;
  }
  [[noreturn]] void fail(const std::string& why) const {
    throw input_error("FASTQ record " + std::to_string(count_) + ": " + why);
  }
  std::istream& in_;
  std::vector<char> buf_ = std::vector<char>(std::size_t(1) << 22);
  std::size_t pos_ = 0, end_ = 0;
  bool eof_ = false;
  std::uint64_t count_ = 0;
};

}  // namespace qgmap
