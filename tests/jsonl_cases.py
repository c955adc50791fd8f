"""JSON-lines impression files for the ingest parity tests (SPEC.md:283 format; the reference's
parse_jsonl_records / record_from_json, serde.hpp:129-170, is the checker). Each case is
(name, bytes): valid files exercise the value semantics, the others one error kind each, placed
after good lines so the reported line number matters."""
import json
import random

GOOD = (b'{"domain":"shop","user_id":"u1","ad_id":"a1","impression_time_ms":1700000000000,'
        b'"features":{"age":31,"ctr":0.0125},"conversions":{"cvr":1700000360000}}')


def rec(**kw):
    r = {"domain": "shop", "user_id": "u", "ad_id": "a", "impression_time_ms": 0, "features": {}, "conversions": {}}
    r.update(kw)
    return json.dumps(r).encode()


def cases():
    c = []
    c.append(("basic", b"\n".join([
        GOOD,
        rec(user_id="user_000042", ad_id="ad_9", impression_time_ms=1700000000000,
            features={"x": -1.5, "y": 2, "z": 1e-7}, conversions={"cvr": 1700000005400, "ctr": 1700000000001}),
        rec(domain="news", features={}, conversions={}),
    ]) + b"\n"))
    c.append(("blank_lines_crlf_no_final_newline",
              b"\n  \t\r\n" + GOOD + b"\r\n\r\n" + rec(user_id="b") + b"\n\n   \n" + rec(user_id="c")))
    c.append(("empty_file", b""))
    c.append(("only_blank", b"\n\n \t \r\n"))
    c.append(("escapes_utf8", b"\n".join([
        b'{"domain":"d\\u00e9","user_id":"q\\"uo\\\\te\\/\\b\\f\\n\\r\\t","ad_id":"\\ud83d\\ude00 emoji",'
        b'"impression_time_ms":5,"features":{"k\\u00e9y":1,"\xc3\xa9t\xc3\xa9":2.5,"\xe2\x82\xac":3},'
        b'"conversions":{"c\\u0076r":7}}',
        '{"domain":"\u65e5\u672c","user_id":"\U0001F600","ad_id":"\u00fc","impression_time_ms":1}'.encode(),
        b'{"domain":"x","user_id":"\\u0000nul","ad_id":"","impression_time_ms":2}',
    ])))
    c.append(("duplicate_keys", b"\n".join([
        b'{"domain":"a","user_id":"first","user_id":"second","ad_id":"x","impression_time_ms":1,'
        b'"impression_time_ms":2,"features":{"f":"str","f":4,"g":1},"features":{"h":5}}',
        b'{"domain":"a","user_id":"u","ad_id":"x","impression_time_ms":1,"conversions":{"t":"bad","t":9,"\\u0074":10}}',
    ])))
    c.append(("number_semantics", b"\n".join([
        b'{"domain":"n","user_id":"u","ad_id":"a","impression_time_ms":18446744073709551615}',
        b'{"domain":"n","user_id":"u","ad_id":"a","impression_time_ms":-9223372036854775808}',
        b'{"domain":"n","user_id":"u","ad_id":"a","impression_time_ms":1.7e12}',
        b'{"domain":"n","user_id":"u","ad_id":"a","impression_time_ms":-2.9}',
        b'{"domain":"n","user_id":"u","ad_id":"a","impression_time_ms":1e300}',
        b'{"domain":"n","user_id":"u","ad_id":"a","impression_time_ms":-9.3e18}',
        b'{"domain":"n","user_id":"u","ad_id":"a","impression_time_ms":-0,"features":{"a":-0.0,"b":-0,'
        b'"c":0.30000000000000004,"d":123456789012345678901234567890,"e":9007199254740993,"f":1.7976931348623158e308,'
        b'"g":-1e-400,"h":4.9406564584124654e-324,"i":2.4703282292062328e-324,"j":-0e5,"k":1.7976931348623157e308,'
        b'"l":2.2250738585072011e-308,"m":18446744073709551616,"n":-9223372036854775809,"o":1E+2,'
        b'"p":0.1e1,"q":100000000000000000000000}}',
        b'{"domain":"n","user_id":"u","ad_id":"a","impression_time_ms":1,"conversions":{"a":1.9,"b":-1.9,'
        b'"c":18446744073709551615,"d":-0.5,"e":1e19,"f":-1e300}}',
    ])))
    c.append(("items_semantics", b"\n".join([
        b'{"domain":"i","user_id":"u","ad_id":"a","impression_time_ms":1,"features":[1,2.5,-3]}',
        b'{"domain":"i","user_id":"u","ad_id":"a","impression_time_ms":1,"features":7.25,"conversions":[10,20,30,40,50,60,70,80,90,100,110]}',
        b'{"domain":"i","user_id":"u","ad_id":"a","impression_time_ms":1,"features":null,"conversions":null}',
        b'{"domain":"i","user_id":"u","ad_id":"a","impression_time_ms":1,"features":{},"conversions":[]}',
        b'{"domain":"i","user_id":"u","ad_id":"a","impression_time_ms":1,"conversions":12}',
    ])))
    c.append(("extra_keys_nesting", b"\n".join([
        b'{"meta":{"a":[1,{"b":[[[]]]},"x\\"}"],"c":null},"domain":"e","user_id":"u","ad_id":"a",'
        b'"impression_time_ms":3,"tags":["x","y"],"score":-1.5e-3,"ok":true}',
        b' \t{ "domain" : "e" , "user_id" : "u" , "ad_id" : "a" , "impression_time_ms" : 4 } \t',
        b'{"domain":"e","user_id":"u","ad_id":"a","impression_time_ms":5,"deep":' + b"[" * 200 + b"]" * 200 + b"}",
    ])))
    c.append(("bom", b"\xef\xbb\xbf" + GOOD + b"\n" + rec(user_id="second")))
    # ---- errors (the first bad line wins)
    c.append(("err_parse_missing_brace", GOOD + b"\n" + GOOD + b"\n" + GOOD[:-1] + b"\n" + GOOD))
    c.append(("err_trailing_content", GOOD + b"\n" + GOOD + b" x\n"))
    c.append(("err_missing_user", GOOD + b'\n{"domain":"d","ad_id":"a","impression_time_ms":1}\n'))
    c.append(("err_missing_ts", GOOD + b'\n{"domain":"d","user_id":"u","ad_id":"a"}\n'))
    c.append(("err_missing_domain_first", b'{"user_id":"u"}\n'))
    c.append(("err_domain_number", GOOD + b'\n{"domain":5,"user_id":"u","ad_id":"a","impression_time_ms":1}\n'))
    c.append(("err_ad_null", GOOD + b'\n{"domain":"d","user_id":"u","ad_id":null,"impression_time_ms":1}\n'))
    c.append(("err_ts_string", b'{"domain":"d","user_id":"u","ad_id":"a","impression_time_ms":"1"}\n'))
    c.append(("err_top_array", GOOD + b"\n[1,2]\n"))
    c.append(("err_top_string", b'"just a string"\n'))
    c.append(("err_feature_string_sorted", GOOD + b'\n' + rec(features={"b": None, "a": "x", "c": 1}) + b"\n"))
    c.append(("err_feature_array_elem", rec(features=[1, "two", None]) + b"\n"))
    c.append(("err_conversion_null", GOOD + b'\n' + rec(conversions={"cvr": None}) + b"\n"))
    c.append(("err_features_string_primitive", rec(features="abc") + b"\n"))
    c.append(("err_invalid_utf8", GOOD + b'\n{"domain":"d\xff","user_id":"u","ad_id":"a","impression_time_ms":1}\n'))
    c.append(("err_overlong_utf8", b'{"domain":"\xc0\xaf","user_id":"u","ad_id":"a","impression_time_ms":1}\n'))
    c.append(("err_surrogate_utf8", b'{"domain":"\xed\xa0\x80","user_id":"u","ad_id":"a","impression_time_ms":1}\n'))
    c.append(("err_lone_surrogate", GOOD + b'\n{"domain":"\\ud800","user_id":"u","ad_id":"a","impression_time_ms":1}\n'))
    c.append(("err_lone_low_surrogate", b'{"domain":"\\udc00x","user_id":"u","ad_id":"a","impression_time_ms":1}\n'))
    c.append(("err_control_char", b'{"domain":"a\tb","user_id":"u","ad_id":"a","impression_time_ms":1}\n'))
    c.append(("err_bad_escape", b'{"domain":"a\\xb","user_id":"u","ad_id":"a","impression_time_ms":1}\n'))
    c.append(("err_bad_literal", GOOD + b'\n{"domain":"d","user_id":"u","ad_id":"a","impression_time_ms":tru}\n'))
    c.append(("err_leading_zero", b'{"domain":"d","user_id":"u","ad_id":"a","impression_time_ms":01}\n'))
    c.append(("err_number_dot", b'{"domain":"d","user_id":"u","ad_id":"a","impression_time_ms":1.}\n'))
    c.append(("err_number_minus", b'{"domain":"d","user_id":"u","ad_id":"a","impression_time_ms":-}\n'))
    c.append(("err_number_exp", b'{"domain":"d","user_id":"u","ad_id":"a","impression_time_ms":1e}\n'))
    c.append(("err_plus_number", b'{"domain":"d","user_id":"u","ad_id":"a","impression_time_ms":+1}\n'))
    c.append(("err_unterminated_string", b'{"domain":"d\n'))
    c.append(("err_only_bom", GOOD + b"\n\xef\xbb\xbf\n"))
    c.append(("err_formfeed_line", GOOD + b"\n\x0c\n"))
    c.append(("err_trailing_comma", b'{"domain":"d","user_id":"u","ad_id":"a","impression_time_ms":1,}\n'))
    c.append(("err_single_quotes", b"{'domain':'d'}\n"))
    c.append(("err_first_of_two", GOOD + b'\n{"domain":"d","ad_id":"a","impression_time_ms":1}\n' + GOOD +
              b"\n{broken\n"))
    c.append(("err_ts_boolean", GOOD + b'\n{"domain":"d","user_id":"u","ad_id":"a","impression_time_ms":true}\n'))
    c.append(("err_feature_boolean", rec(features={"a": 1, "b": True}) + b"\n"))
    c.append(("err_conversions_boolean", rec(conversions=False) + b"\n"))
    c.append(("err_overflow_ts", GOOD + b'\n{"domain":"d","user_id":"u","ad_id":"a","impression_time_ms":1e400}\n'))
    c.append(("err_overflow_ignored_key", b'{"x":{"y":[-2e999]},"domain":"d","user_id":5,,}\n'))
    c.append(("err_syntax_before_overflow", b'{"domain":"d",,"x":1e999}\n'))
    c.append(("err_overflow_long_integer", GOOD + b"\n" + rec(features={"big": 1}).replace(b'"big": 1', b'"big": ' + b"9" * 400) + b"\n"))
    c.append(("err_two_values", b'{"domain":"d","user_id":"u","ad_id":"a","impression_time_ms":1} {}\n'))
    return c


def random_file(n, seed, tasks=("cvr", "ctr", "atc")):
    """n impression records of the shape the Zipper consumes (random users/ads/timestamps,
    17-digit feature values, conversions on a subset of tasks), as one JSONL file."""
    rng = random.Random(seed)
    lines = []
    for i in range(n):
        ts = 1_700_000_000_000 + 37 * i
        feats = {f"f{k}": rng.choice([rng.uniform(-1e6, 1e6), rng.random(), float(rng.randint(-100, 100)),
                                      rng.uniform(-1, 1) * 10 ** rng.randint(-300, 300)])
                 for k in range(rng.randint(0, 8))}
        convs = {t: ts + rng.randint(0, 8 * 86_400_000) for t in tasks if rng.random() < 0.3}
        r = {"domain": f"d{rng.randint(0, 15)}", "user_id": f"u{rng.randint(0, 10**8)}",
             "ad_id": f"a{rng.randint(0, 10**6)}", "impression_time_ms": ts, "features": feats,
             "conversions": convs}
        lines.append(json.dumps(r, separators=(",", ":"), ensure_ascii=rng.random() < 0.5))
        if rng.random() < 0.01:
            lines.append("")
    return ("\n".join(lines) + "\n").encode()
