"""Golden fixtures for the dataset file format, made by RUNNING THE REFERENCE's reader and
writer (reference cli.py:47-75, model.py:174-197) on crafted CSV files.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_ingest_golden.py

Writes tests/golden/csv/*.csv (the inputs) and tests/golden/csv/expected.json +
csv_*.npz: for every file either the Dataset arrays the reference's read_dataset_csv
returns (and, for written files, the bytes its write_dataset_csv produces) or the
exception class and message it raises ("{path}" stands for the file path).
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "csv")

sys.path.insert(0, "/root/reference/pkg/src")
from tissuemix import cli, model  # noqa: E402  (the reference)
from tissuemix.samplers import RngStream  # noqa: E402


def hand_files():
    """Crafted inputs: formats the reference accepts beyond repr(), and every error kind."""
    f = {}
    f["mixed_formats.csv"] = (
        "r,d_1,d_2,d_3\n"
        "0.5,1,0,1\n"
        " 1.25 ,0.0,1.0,0\n"
        "+.5,1.,0,1\n"
        "-3.0e-5,1e0,0E+0,1\n"
        "1_000.5,0,1,0\n"
        "1e-320,0.1,0.2,0.7\n"
        "2.4703282292062328e-324,1,1,1\n"
        "123456789012345678901234567890,0,0,0\n"
        "0.1000000000000000055511151231257827021181583404541015625,1,0,0\n"
        "9007199254740993,0,1,0\n"
        "1.7976931348623157e308,0,0,1\n"
        "\"0.75\",\"1\",0,1\n"
        "\t-0.0\t,0,0,1\n"
        "3.141592653589793238462643383279,0.333333333333333333333333,0.25,0.125\n"
    )
    f["crlf_blank.csv"] = "r,d_1,d_2\r\n0.5,1,0\r\n\r\n1.5,0,1\r\n\n-2.25,1,1"
    f["no_trailing_newline.csv"] = "r,d_1,d_2\n0.1,1,0\n0.2,0,1"
    # errors
    f["err_header.csv"] = "x,d_1,d_2\n0.1,1,0\n"
    f["err_header_short.csv"] = "r,d_1\n0.1,1\n"
    f["err_empty.csv"] = ""
    f["err_blank_header.csv"] = "\nr,d_1,d_2\n0.1,1,0\n"
    f["err_no_records.csv"] = "r,d_1,d_2\n\n\n"
    f["err_fields.csv"] = "r,d_1,d_2\n0.1,1,0\n0.2,1\n0.3,1,0\n"
    f["err_fields_long.csv"] = "r,d_1,d_2\n0.1,1,0\n0.2,1,0,1\n"
    f["err_parse_r.csv"] = "r,d_1,d_2\n0.1,1,0\nabc,1,0\n0.3,1\n"
    f["err_parse_d.csv"] = "r,d_1,d_2\n0.1,1,0\n0.2,1,0x10\n"
    f["err_first_wins.csv"] = "r,d_1,d_2\n0.1,1,0\n0.2,1\n0.3,zz,0\n"
    f["err_nan_d.csv"] = "r,d_1,d_2\n0.1,1,0\n0.2,nan,0\n"
    f["err_inf_r.csv"] = "r,d_1,d_2\n0.1,1,0\n-Infinity,1,0\n"
    f["err_inf_r_nan_d.csv"] = "r,d_1,d_2\ninf,1,nan\n"
    f["err_bad_r_nan_d.csv"] = "r,d_1,d_2\n1..2,1,nan\n"
    f["err_underscore.csv"] = "r,d_1,d_2\n1__0,1,0\n"
    f["err_ws_only_row.csv"] = "r,d_1,d_2\n0.1,1,0\n   \n"
    # csv.reader quoting (the GPU reader hands any file with a quote to the host reader)
    f["quoted_fields.csv"] = ('"r","d_1","d_2"\n"0.5","1","0"\n"1.5",0,"1"\n"2.5\n",1,0\n'
                              '"-1.25" ,1,0\n\n"3"e0,0,1\r\n4.5,"1","0"\r\n"7.0",1,"1\n"\n')
    f["err_quoted_comma.csv"] = 'r,d_1,d_2\n0.1,1,0\n"1,5",1,0\n'
    f["err_quoted_fields.csv"] = 'r,d_1,d_2\n0.1,"1,0"\n'
    f["err_doubled_quote.csv"] = 'r,d_1,d_2\n"1""0",1,0\n'
    f["err_quote_in_field.csv"] = "r,d_1,d_2\n0.5,1,0\n0.25,x'\"y,0\n"
    f["err_quoted_header.csv"] = '"r,d_1",d_2\n0.1,1\n'
    return f


def written_datasets():
    """Datasets the reference WRITES (cli.py:47-56): synth output and real-valued profiles."""
    out = {}
    rng = RngStream(56)
    truth = model.ModelParams(K=np.array([0.65, 0.28]), Lam=np.linalg.inv(model.REFERENCE_LAMBDA_INV), rho=5.0)
    out["w_mock56.csv"] = model.synth_generate(rng, truth, model.random_profiles(rng, 56, 3))
    rng = RngStream(34)
    raw = rng.uniforms(300 * 4).reshape(300, 4)
    profiles = [model.ExpressionProfile(row) for row in raw]
    truth = model.ModelParams(K=np.array([0.1, 0.2, 0.3]), Lam=100.0 * np.eye(3), rho=50.0)
    out["w_real300_n4.csv"] = model.synth_generate(rng, truth, profiles)
    rng = RngStream(7)
    truth = model.ModelParams(K=np.full(7, 0.1), Lam=100.0 * np.eye(7), rho=1e6)
    out["w_n8_2000.csv"] = model.synth_generate(rng, truth, model.random_profiles(rng, 2000, 8))
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    expected = {}
    for name, text in hand_files().items():
        with open(os.path.join(OUT, name), "w", newline="", encoding="utf-8") as fh:
            fh.write(text)
    for name, ds in written_datasets().items():
        cli.write_dataset_csv(os.path.join(OUT, name), ds)
    for name in sorted(os.listdir(OUT)):
        if not name.endswith(".csv"):
            continue
        path = os.path.join(OUT, name)
        try:
            ds = cli.read_dataset_csv(path)
        except Exception as e:  # noqa: BLE001
            expected[name] = {"error": type(e).__name__, "message": str(e).replace(path, "{path}")}
            continue
        np.savez(os.path.join(OUT, name[:-4] + ".npz"), r=ds.r, mu=ds.mu, D=ds.D, n_networks=ds.n_networks)
        back = path + ".back"
        cli.write_dataset_csv(back, ds)  # the reference writer's bytes for this dataset
        os.replace(back, os.path.join(OUT, name[:-4] + ".written"))
        expected[name] = {"V": int(ds.V), "n_networks": int(ds.n_networks)}
    with open(os.path.join(OUT, "expected.json"), "w") as fh:
        json.dump(expected, fh, indent=1, sort_keys=True)
    for k, v in sorted(expected.items()):
        print(k, v)


if __name__ == "__main__":
    main()
