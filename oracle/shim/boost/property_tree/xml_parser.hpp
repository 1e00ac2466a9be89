// oracle/shim/boost/property_tree/xml_parser.hpp — read_xml for the
// Boost.PropertyTree shim (oracle/_ref only).  Elements become children keyed
// by tag name in document order, attributes go under "<xmlattr>", text goes
// to the node's data; the XML declaration, comments, processing instructions
// and DOCTYPE are skipped; the five predefined entities and numeric
// character references are decoded.  Malformed input throws
// xml_parser_error, as Boost does.
#pragma once

#include <cctype>
#include <fstream>
#include <sstream>
#include <string>

#include "ptree.hpp"

namespace boost {
namespace property_tree {

class xml_parser_error : public ptree_error {
 public:
  using ptree_error::ptree_error;
};

namespace xml_parser {
namespace detail {

inline std::string decode(const std::string& s) {
  std::string out;
  for (std::size_t i = 0; i < s.size(); ++i) {
    if (s[i] != '&') {
      out += s[i];
      continue;
    }
    std::size_t semi = s.find(';', i);
    if (semi == std::string::npos) throw xml_parser_error("unterminated entity");
    std::string ent = s.substr(i + 1, semi - i - 1);
    if (ent == "lt") out += '<';
    else if (ent == "gt") out += '>';
    else if (ent == "amp") out += '&';
    else if (ent == "quot") out += '"';
    else if (ent == "apos") out += '\'';
    else if (!ent.empty() && ent[0] == '#') {
      unsigned long cp = (ent.size() > 1 && (ent[1] == 'x' || ent[1] == 'X'))
                             ? std::stoul(ent.substr(2), nullptr, 16)
                             : std::stoul(ent.substr(1), nullptr, 10);
      if (cp < 0x80) {
        out += static_cast<char>(cp);
      } else if (cp < 0x800) {
        out += static_cast<char>(0xC0 | (cp >> 6));
        out += static_cast<char>(0x80 | (cp & 0x3F));
      } else {
        out += static_cast<char>(0xE0 | (cp >> 12));
        out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
        out += static_cast<char>(0x80 | (cp & 0x3F));
      }
    } else {
      throw xml_parser_error("unknown entity &" + ent + ";");
    }
    i = semi;
  }
  return out;
}

struct Parser {
  const std::string& s;
  std::size_t i = 0;
  void fail(const std::string& what) { throw xml_parser_error("xml parse error: " + what); }
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  bool starts(const char* p) const { return s.compare(i, std::char_traits<char>::length(p), p) == 0; }
  void skip_until(const char* end) {
    std::size_t e = s.find(end, i);
    if (e == std::string::npos) fail(std::string("missing ") + end);
    i = e + std::char_traits<char>::length(end);
  }
  // Skips declarations, comments, PIs, DOCTYPE; returns true if something was skipped.
  bool skip_misc() {
    if (starts("<?")) {
      skip_until("?>");
      return true;
    }
    if (starts("<!--")) {
      skip_until("-->");
      return true;
    }
    if (starts("<!DOCTYPE")) {
      skip_until(">");
      return true;
    }
    return false;
  }
  std::string name() {
    std::size_t b = i;
    while (i < s.size() && (std::isalnum(static_cast<unsigned char>(s[i])) || s[i] == '_' ||
                            s[i] == '-' || s[i] == ':' || s[i] == '.'))
      ++i;
    if (i == b) fail("expected a name");
    return s.substr(b, i - b);
  }
  void element(ptree& parent) {
    if (s[i] != '<') fail("expected '<'");
    ++i;
    std::string tag = name();
    ptree node;
    ptree attrs;
    bool has_attrs = false;
    for (;;) {
      ws();
      if (i >= s.size()) fail("unterminated tag <" + tag + ">");
      if (starts("/>")) {
        i += 2;
        if (has_attrs) node.push_back_child("<xmlattr>", attrs);
        parent.push_back_child(tag, std::move(node));
        return;
      }
      if (s[i] == '>') {
        ++i;
        break;
      }
      std::string an = name();
      ws();
      if (i >= s.size() || s[i] != '=') fail("expected '=' after attribute " + an);
      ++i;
      ws();
      if (i >= s.size() || (s[i] != '"' && s[i] != '\'')) fail("expected quoted attribute value");
      char q = s[i++];
      std::size_t e = s.find(q, i);
      if (e == std::string::npos) fail("unterminated attribute value");
      attrs.push_back_child(an, ptree(decode(s.substr(i, e - i))));
      has_attrs = true;
      i = e + 1;
    }
    if (has_attrs) node.push_back_child("<xmlattr>", attrs);
    std::string text;
    for (;;) {
      if (i >= s.size()) fail("unterminated element <" + tag + ">");
      if (starts("</")) {
        i += 2;
        std::string close = name();
        if (close != tag) fail("mismatched </" + close + "> for <" + tag + ">");
        ws();
        if (i >= s.size() || s[i] != '>') fail("expected '>'");
        ++i;
        break;
      }
      if (starts("<![CDATA[")) {
        i += 9;
        std::size_t e = s.find("]]>", i);
        if (e == std::string::npos) fail("unterminated CDATA");
        text += s.substr(i, e - i);
        i = e + 3;
        continue;
      }
      if (skip_misc()) continue;
      if (s[i] == '<') {
        element(node);
        continue;
      }
      std::size_t e = s.find('<', i);
      if (e == std::string::npos) e = s.size();
      text += decode(s.substr(i, e - i));
      i = e;
    }
    node.data() = text;
    parent.push_back_child(tag, std::move(node));
  }
  void document(ptree& root) {
    for (;;) {
      ws();
      if (i >= s.size()) break;
      if (skip_misc()) continue;
      if (s[i] == '<') {
        element(root);
        continue;
      }
      fail("text outside the root element");
    }
    if (root.empty()) fail("no root element");
  }
};

}  // namespace detail

inline void read_xml(std::istream& in, ptree& pt, int flags = 0) {
  (void)flags;
  std::stringstream ss;
  ss << in.rdbuf();
  std::string text = ss.str();
  ptree out;
  detail::Parser p{text};
  p.document(out);
  pt = std::move(out);
}

inline void read_xml(const std::string& path, ptree& pt, int flags = 0) {
  std::ifstream f(path);
  if (!f) throw xml_parser_error(path + ": cannot open file");
  read_xml(f, pt, flags);
}

}  // namespace xml_parser

using xml_parser::read_xml;

}  // namespace property_tree
}  // namespace boost
