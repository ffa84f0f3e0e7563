// Minimal YAML reader for the scenario-v1 subset.
//
// The reference parses scenarios with yaml-cpp (`/root/reference/proj/src/scenario.cpp:322-374`);
// yaml-cpp is not available to this engine, and the scenario files only use a small subset of
// YAML: block mappings and sequences, flow mappings `{k: v, ...}` and flow sequences `[a, b]`,
// `#` comments, plain and quoted scalars.  Scalars are kept as text; typing happens in the
// loader with yaml-cpp's `as<T>()` conversion rules.  Every node carries its 1-based line so
// errors can say "file:line" like `scenario.cpp:100-106`.
#pragma once

#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace mgb::yaml {

struct Node {
    enum Kind { kNull, kScalar, kMap, kSeq } kind = kNull;
    int line = 1;
    std::string text;                                                 // scalar
    std::vector<std::pair<std::string, std::shared_ptr<Node>>> map;  // insertion order
    std::vector<int> key_lines;
    std::vector<std::shared_ptr<Node>> seq;

    const Node* get(const std::string& k) const {
        for (const auto& kv : map)
            if (kv.first == k) return kv.second.get();
        return nullptr;
    }
    int key_line(const std::string& k) const {
        for (size_t i = 0; i < map.size(); ++i)
            if (map[i].first == k) return key_lines[i];
        return line;
    }
};

struct ParseError : std::runtime_error {
    int line;
    ParseError(const std::string& m, int l) : std::runtime_error(m), line(l) {}
};

namespace detail {

struct Line {
    int indent;
    std::string text;
    int no;
};

inline std::string strip_comment(const std::string& s) {
    bool sq = false, dq = false;
    for (size_t i = 0; i < s.size(); ++i) {
        const char c = s[i];
        if (c == '\'' && !dq) sq = !sq;
        else if (c == '"' && !sq) dq = !dq;
        else if (c == '#' && !sq && !dq && (i == 0 || s[i - 1] == ' ' || s[i - 1] == '\t')) return s.substr(0, i);
    }
    return s;
}

inline std::string trim(const std::string& s) {
    size_t a = 0, b = s.size();
    while (a < b && (s[a] == ' ' || s[a] == '\t' || s[a] == '\r')) ++a;
    while (b > a && (s[b - 1] == ' ' || s[b - 1] == '\t' || s[b - 1] == '\r')) --b;
    return s.substr(a, b - a);
}

inline std::string unquote(const std::string& s, int line) {
    if (s.size() >= 2 && ((s.front() == '"' && s.back() == '"') || (s.front() == '\'' && s.back() == '\''))) {
        std::string out;
        const bool dq = s.front() == '"';
        for (size_t i = 1; i + 1 < s.size(); ++i) {
            char c = s[i];
            if (dq && c == '\\' && i + 2 < s.size()) {
                const char n = s[++i];
                c = n == 'n' ? '\n' : n == 't' ? '\t' : n;
            } else if (!dq && c == '\'' && i + 2 < s.size() && s[i + 1] == '\'') {
                ++i;
            }
            out += c;
        }
        return out;
    }
    (void)line;
    return s;
}

// Find the ':' that separates a mapping key from its value (outside quotes/brackets).
inline size_t find_colon(const std::string& s) {
    bool sq = false, dq = false;
    int depth = 0;
    for (size_t i = 0; i < s.size(); ++i) {
        const char c = s[i];
        if (c == '\'' && !dq) sq = !sq;
        else if (c == '"' && !sq) dq = !dq;
        else if (!sq && !dq) {
            if (c == '[' || c == '{') ++depth;
            else if (c == ']' || c == '}') --depth;
            else if (c == ':' && depth == 0 && (i + 1 == s.size() || s[i + 1] == ' ' || s[i + 1] == '\t')) return i;
        }
    }
    return std::string::npos;
}

class FlowParser {
public:
    FlowParser(const std::string& s, int line) : s_(s), line_(line) {}
    std::shared_ptr<Node> parse() {
        auto n = value();
        ws();
        if (i_ != s_.size()) throw ParseError("unexpected trailing characters in flow collection", line_);
        return n;
    }

private:
    void ws() {
        while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t')) ++i_;
    }
    std::shared_ptr<Node> value() {
        ws();
        if (i_ >= s_.size()) throw ParseError("unexpected end of flow collection", line_);
        auto n = std::make_shared<Node>();
        n->line = line_;
        if (s_[i_] == '{') {
            ++i_;
            n->kind = Node::kMap;
            ws();
            if (i_ < s_.size() && s_[i_] == '}') {
                ++i_;
                return n;
            }
            for (;;) {
                std::string k = scalar_text(true);
                ws();
                if (i_ >= s_.size() || s_[i_] != ':') throw ParseError("expected ':' in flow mapping", line_);
                ++i_;
                auto v = value();
                n->map.emplace_back(unquote(trim(k), line_), v);
                n->key_lines.push_back(line_);
                ws();
                if (i_ < s_.size() && s_[i_] == ',') {
                    ++i_;
                    continue;
                }
                if (i_ < s_.size() && s_[i_] == '}') {
                    ++i_;
                    return n;
                }
                throw ParseError("expected ',' or '}' in flow mapping", line_);
            }
        }
        if (s_[i_] == '[') {
            ++i_;
            n->kind = Node::kSeq;
            ws();
            if (i_ < s_.size() && s_[i_] == ']') {
                ++i_;
                return n;
            }
            for (;;) {
                n->seq.push_back(value());
                ws();
                if (i_ < s_.size() && s_[i_] == ',') {
                    ++i_;
                    continue;
                }
                if (i_ < s_.size() && s_[i_] == ']') {
                    ++i_;
                    return n;
                }
                throw ParseError("expected ',' or ']' in flow sequence", line_);
            }
        }
        n->kind = Node::kScalar;
        n->text = unquote(trim(scalar_text(false)), line_);
        return n;
    }
    std::string scalar_text(bool is_key) {
        ws();
        size_t start = i_;
        if (i_ < s_.size() && (s_[i_] == '"' || s_[i_] == '\'')) {
            const char q = s_[i_++];
            while (i_ < s_.size() && s_[i_] != q) {
                if (q == '"' && s_[i_] == '\\') ++i_;
                ++i_;
            }
            ++i_;
            return s_.substr(start, i_ - start);
        }
        while (i_ < s_.size()) {
            const char c = s_[i_];
            if (c == ',' || c == '}' || c == ']') break;
            if (is_key && c == ':') break;
            ++i_;
        }
        return s_.substr(start, i_ - start);
    }
    const std::string& s_;
    size_t i_ = 0;
    int line_;
};

class BlockParser {
public:
    explicit BlockParser(std::vector<Line> lines) : L_(std::move(lines)) {}

    std::shared_ptr<Node> parse_document() {
        if (L_.empty()) return std::make_shared<Node>();
        auto n = block(L_[0].indent);
        if (p_ != L_.size()) throw ParseError("unexpected indentation", L_[p_].no);
        return n;
    }

private:
    static bool is_seq_item(const std::string& t) { return t == "-" || (t.size() >= 2 && t[0] == '-' && t[1] == ' '); }

    std::shared_ptr<Node> inline_value(const std::string& v, int line) {
        const std::string t = trim(v);
        if (!t.empty() && (t[0] == '{' || t[0] == '[')) return FlowParser(t, line).parse();
        auto n = std::make_shared<Node>();
        n->kind = Node::kScalar;
        n->line = line;
        n->text = unquote(t, line);
        return n;
    }

    std::shared_ptr<Node> block(int indent) {
        if (is_seq_item(L_[p_].text)) return sequence(indent);
        return mapping(indent);
    }

    std::shared_ptr<Node> sequence(int indent) {
        auto n = std::make_shared<Node>();
        n->kind = Node::kSeq;
        n->line = L_[p_].no;
        while (p_ < L_.size() && L_[p_].indent == indent && is_seq_item(L_[p_].text)) {
            Line& cur = L_[p_];
            const std::string rest = cur.text.size() > 1 ? cur.text.substr(2) : std::string();
            const std::string rt = trim(rest);
            if (rt.empty()) {
                ++p_;
                if (p_ < L_.size() && L_[p_].indent > indent) n->seq.push_back(block(L_[p_].indent));
                else n->seq.push_back(std::make_shared<Node>());
                continue;
            }
            if (rt[0] != '{' && rt[0] != '[' && find_colon(rt) != std::string::npos) {
                // "- key: value": a mapping whose first key sits at indent + 2 + leading spaces
                size_t lead = 0;
                while (lead < rest.size() && rest[lead] == ' ') ++lead;
                cur.indent = indent + 2 + static_cast<int>(lead);
                cur.text = rest.substr(lead);
                n->seq.push_back(mapping(cur.indent));
                continue;
            }
            n->seq.push_back(inline_value(rt, cur.no));
            ++p_;
        }
        return n;
    }

    std::shared_ptr<Node> mapping(int indent) {
        auto n = std::make_shared<Node>();
        n->kind = Node::kMap;
        n->line = L_[p_].no;
        while (p_ < L_.size() && L_[p_].indent == indent) {
            const Line cur = L_[p_];
            if (is_seq_item(cur.text)) throw ParseError("sequence item where a mapping key was expected", cur.no);
            const size_t c = find_colon(cur.text);
            if (c == std::string::npos) throw ParseError("expected 'key: value'", cur.no);
            const std::string key = unquote(trim(cur.text.substr(0, c)), cur.no);
            const std::string val = trim(cur.text.substr(c + 1));
            for (const auto& kv : n->map)
                if (kv.first == key) throw ParseError("duplicate key '" + key + "'", cur.no);
            ++p_;
            std::shared_ptr<Node> v;
            if (!val.empty()) {
                v = inline_value(val, cur.no);
            } else if (p_ < L_.size() && (L_[p_].indent > indent || (L_[p_].indent == indent && is_seq_item(L_[p_].text)))) {
                v = block(L_[p_].indent);
            } else {
                v = std::make_shared<Node>();
                v->line = cur.no;
            }
            n->map.emplace_back(key, v);
            n->key_lines.push_back(cur.no);
        }
        if (p_ < L_.size() && L_[p_].indent > indent) throw ParseError("unexpected indentation", L_[p_].no);
        return n;
    }

    std::vector<Line> L_;
    size_t p_ = 0;
};

}  // namespace detail

// Parse a YAML document (scenario subset). Throws ParseError with a 1-based line.
inline std::shared_ptr<Node> parse(const std::string& text) {
    std::vector<detail::Line> lines;
    size_t pos = 0;
    int no = 0;
    while (pos <= text.size()) {
        size_t e = text.find('\n', pos);
        if (e == std::string::npos) e = text.size();
        std::string raw = text.substr(pos, e - pos);
        ++no;
        pos = e + 1;
        for (char ch : raw)
            if (ch == '\t') throw ParseError("tab characters are not allowed in indentation", no);
        std::string s = detail::strip_comment(raw);
        const std::string t = detail::trim(s);
        if (t.empty() || t == "---" || t == "...") {
            if (e == text.size()) break;
            continue;
        }
        int ind = 0;
        while (ind < static_cast<int>(s.size()) && s[ind] == ' ') ++ind;
        lines.push_back({ind, t, no});
        if (e == text.size()) break;
    }
    return detail::BlockParser(std::move(lines)).parse_document();
}

}  // namespace mgb::yaml
